// io.cu -- the reference's file containers on the device path (SURVEY 8f,
// rank 3): FMAT1 feature matrices, CSR1 graphs and text edge lists
// (io.hpp:25-41, io.cpp:83-207).
//
// Layouts (little-endian, io.hpp:31-38):
//   FMAT1  "FMAT1" | u64 rows | u64 dim | rows * dim float32
//   CSR1   "CSR1"  | u8 orientation (0 src-major, else dst-major)
//          | u64 num_rows | u64 num_cols | u64 num_edges
//          | (num_rows + 1) u64 indptr | num_edges u64 indices
//          | num_edges u64 edge_ids
//
// Device loaders stream the file through a two-slot pinned ring: the pread
// of chunk k + 1 overlaps the DMA of chunk k.  A CSR1 payload's 64-bit
// elements are narrowed to the 32-bit ids of the device CSR by a kernel
// (k_narrow, with an overflow flag: io.cpp:71-73), then checked on the
// device with the reference's validate() rules and messages
// (csr.cpp:111-156) before the handle is built.  Host readers / writers
// serve the C++ shim and the tests.  Errors: GSPMM_ERR_IO (IoError) and
// GSPMM_ERR_PARSE (ParseError, with the line number), error.hpp:37-45.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <string_view>
#include <vector>

#include "gspmm_b200.h"
#include "internal.h"

namespace gspmm_b200 {
namespace {

constexpr size_t kChunkBytes = 32u << 20;  // one ring slot

int io_fail(const std::string& msg) { return set_last_error(GSPMM_ERR_IO, msg); }
int cuda_io_fail(cudaError_t e, const char* where) {
  return set_last_error(GSPMM_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// A read-only file with exact-length positional reads.
struct InFile {
  int fd = -1;
  std::string path;
  uint64_t size = 0;
  explicit InFile(const char* p) : path(p ? p : "") {
    if (!p) return;
    fd = ::open(p, O_RDONLY);
    if (fd >= 0) {
      struct stat st;
      if (::fstat(fd, &st) == 0 && S_ISREG(st.st_mode)) {
        size = static_cast<uint64_t>(st.st_size);
      } else {
        ::close(fd);
        fd = -1;
      }
    }
  }
  ~InFile() {
    if (fd >= 0) ::close(fd);
  }
  bool ok() const { return fd >= 0; }
  // false when fewer than n bytes remain at off
  bool read(void* dst, size_t n, uint64_t off) const {
    char* p = static_cast<char*>(dst);
    while (n) {
      const ssize_t got = ::pread(fd, p, n, static_cast<off_t>(off));
      if (got < 0 && errno == EINTR) continue;
      if (got <= 0) return false;
      p += got;
      off += static_cast<uint64_t>(got);
      n -= static_cast<size_t>(got);
    }
    return true;
  }
};

struct OutFile {
  FILE* f = nullptr;
  std::string path;
  explicit OutFile(const char* p) : path(p ? p : "") {
    if (p) f = std::fopen(p, "wb");
  }
  ~OutFile() {
    if (f) std::fclose(f);
  }
  bool write(const void* src, size_t n) { return n == 0 || std::fwrite(src, 1, n, f) == n; }
  bool close() {
    const bool ok = std::fclose(f) == 0;
    f = nullptr;
    return ok;
  }
};

struct Fmat1Header {
  int64_t rows = 0, dim = 0;
  static constexpr uint64_t kBytes = 5 + 16;
};

int read_fmat1_header(const InFile& in, Fmat1Header* h) {
  if (!in.ok()) return io_fail("cannot open " + in.path);
  unsigned char raw[Fmat1Header::kBytes];
  if (!in.read(raw, 5, 0) || std::memcmp(raw, "FMAT1", 5) != 0)
    return io_fail(in.path + ": not a FMAT1 file");
  if (!in.read(raw + 5, 16, 5)) return io_fail(in.path + ": truncated file");
  uint64_t r, d;
  std::memcpy(&r, raw + 5, 8);
  std::memcpy(&d, raw + 13, 8);
  h->rows = static_cast<int64_t>(r);
  h->dim = static_cast<int64_t>(d);
  if (h->rows < 0 || h->dim < 0) return io_fail(in.path + ": bad dimensions");
  // rows * dim floats must be present (io.cpp:160-163)
  const unsigned __int128 need = static_cast<unsigned __int128>(r) * d * 4u;
  if (need > in.size - Fmat1Header::kBytes) return io_fail(in.path + ": truncated data section");
  return GSPMM_OK;
}

struct Csr1Header {
  int orientation = GSPMM_DST_MAJOR;
  uint64_t rows = 0, cols = 0, edges = 0;
  static constexpr uint64_t kBytes = 4 + 1 + 24;
  uint64_t indptr_off() const { return kBytes; }
  uint64_t indices_off() const { return kBytes + 8 * (rows + 1); }
  uint64_t eids_off() const { return indices_off() + 8 * edges; }
};

int read_csr1_header(const InFile& in, Csr1Header* h) {
  if (!in.ok()) return io_fail("cannot open " + in.path);
  unsigned char raw[Csr1Header::kBytes];
  if (!in.read(raw, 4, 0) || std::memcmp(raw, "CSR1", 4) != 0)
    return io_fail(in.path + ": not a CSR1 file");
  if (!in.read(raw + 4, 25, 4)) return io_fail(in.path + ": truncated file");
  h->orientation = raw[4] ? GSPMM_DST_MAJOR : GSPMM_SRC_MAJOR;
  std::memcpy(&h->rows, raw + 5, 8);
  std::memcpy(&h->cols, raw + 13, 8);
  std::memcpy(&h->edges, raw + 21, 8);
  constexpr uint64_t cap = std::numeric_limits<uint32_t>::max();
  if (h->rows > cap || h->cols > cap || h->edges > cap)
    return io_fail(in.path + ": id does not fit the configured id width");
  const unsigned __int128 need =
      static_cast<unsigned __int128>(8) * (h->rows + 1) + static_cast<unsigned __int128>(16) * h->edges;
  if (need > in.size - Csr1Header::kBytes) return io_fail(in.path + ": truncated file");
  return GSPMM_OK;
}

// u64 file elements -> u32 host ids (read_u64_array, io.cpp:65-76)
int read_u64_as_u32(const InFile& in, uint64_t off, uint64_t count, uint32_t* dst) {
  std::vector<uint64_t> buf(std::min<uint64_t>(count, kChunkBytes / 8));
  for (uint64_t done = 0; done < count;) {
    const uint64_t n = std::min<uint64_t>(buf.size(), count - done);
    if (!in.read(buf.data(), n * 8, off + done * 8)) return io_fail(in.path + ": truncated file");
    for (uint64_t i = 0; i < n; ++i) {
      if (buf[i] > std::numeric_limits<uint32_t>::max())
        return io_fail(in.path + ": id does not fit the configured id width");
      dst[done + i] = static_cast<uint32_t>(buf[i]);
    }
    done += n;
  }
  return GSPMM_OK;
}

// ---- device side -----------------------------------------------------------

__global__ void k_narrow(const uint64_t* __restrict__ src, uint64_t n, uint32_t* __restrict__ dst,
                         uint32_t* __restrict__ overflow) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  bool bad = false;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t v = src[i];
    bad |= (v >> 32) != 0;
    dst[i] = static_cast<uint32_t>(v);
  }
  if (bad) *overflow = 1u;
}

// validate(), csr.cpp:128-153, one kernel per rule; each reports the LOWEST
// offending nonzero through an atomicMin, which is the one the reference's
// sequential scan stops at.
__global__ void k_check_range(const uint32_t* __restrict__ indices, uint64_t m, uint32_t num_cols,
                              unsigned long long* __restrict__ bad) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < m; j += stride)
    if (indices[j] >= num_cols) {
      atomicMin(bad, static_cast<unsigned long long>(j));
      return;
    }
}

// first[e] = lowest nonzero carrying edge id e
__global__ void k_first_use(const uint32_t* __restrict__ eids, uint64_t m, uint32_t* __restrict__ first) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < m; j += stride) {
    const uint32_t e = eids[j];
    if (e < m) atomicMin(first + e, static_cast<uint32_t>(j));
  }
}

// nonzero j breaks the permutation when its id is out of range or was used
// by an earlier nonzero ("seen", csr.cpp:136-142)
__global__ void k_check_perm(const uint32_t* __restrict__ eids, uint64_t m,
                             const uint32_t* __restrict__ first, unsigned long long* __restrict__ bad) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < m; j += stride) {
    const uint32_t e = eids[j];
    if (e >= m || first[e] != static_cast<uint32_t>(j)) {
      atomicMin(bad, static_cast<unsigned long long>(j));
      return;
    }
  }
}

__global__ void k_mark_row_starts(const uint32_t* __restrict__ indptr, uint32_t rows, uint64_t m,
                                  uint32_t* __restrict__ start_bits) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += stride) {
    const uint32_t j = indptr[r];
    if (j < m) atomicOr(start_bits + (j >> 5), 1u << (j & 31));
  }
}

// (neighbour, edge id) strictly ascending inside each row (csr.cpp:143-153)
__global__ void k_check_sorted(const uint32_t* __restrict__ indices, const uint32_t* __restrict__ eids,
                               uint64_t m, const uint32_t* __restrict__ start_bits,
                               unsigned long long* __restrict__ bad) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j + 1 < m; j += stride) {
    const uint64_t k = j + 1;
    if ((start_bits[k >> 5] >> (k & 31)) & 1u) continue;  // k opens a row
    const uint32_t a = indices[j], b = indices[k];
    if (!(a < b || (a == b && eids[j] < eids[k]))) {
      atomicMin(bad, static_cast<unsigned long long>(k));
      return;
    }
  }
}

constexpr int kGrid = 148 * 8, kBlock = 256;

// The two-slot pinned ring of a device loader.
struct Ring {
  void* host[2] = {nullptr, nullptr};
  void* dev[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  bool busy[2] = {false, false};
  cudaError_t init(bool device_stage) {
    for (int k = 0; k < 2; ++k) {
      cudaError_t e = cudaMallocHost(&host[k], kChunkBytes);
      if (e) return e;
      if (device_stage && (e = cudaMalloc(&dev[k], kChunkBytes))) return e;
      if ((e = cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming))) return e;
    }
    return cudaSuccess;
  }
  cudaError_t acquire(int k) {
    if (!busy[k]) return cudaSuccess;
    busy[k] = false;
    return cudaEventSynchronize(ev[k]);
  }
  cudaError_t release(int k, cudaStream_t s) {
    busy[k] = true;
    return cudaEventRecord(ev[k], s);
  }
  ~Ring() {
    for (int k = 0; k < 2; ++k) {
      if (ev[k]) {
        cudaEventSynchronize(ev[k]);
        cudaEventDestroy(ev[k]);
      }
      if (host[k]) cudaFreeHost(host[k]);
      if (dev[k]) cudaFree(dev[k]);
    }
  }
};

// count u64 file elements at off -> d_dst[count] u32, through the ring
int stream_u64_to_device(const InFile& in, uint64_t off, uint64_t count, uint32_t* d_dst, Ring& ring,
                         uint32_t* d_overflow, cudaStream_t s) {
  const uint64_t per = kChunkBytes / 8;
  int slot = 0;
  for (uint64_t done = 0; done < count; slot ^= 1) {
    const uint64_t n = std::min<uint64_t>(per, count - done);
    cudaError_t e = ring.acquire(slot);
    if (e) return cuda_io_fail(e, "csr1 ring");
    if (!in.read(ring.host[slot], n * 8, off + done * 8)) return io_fail(in.path + ": truncated file");
    if ((e = cudaMemcpyAsync(ring.dev[slot], ring.host[slot], n * 8, cudaMemcpyHostToDevice, s)))
      return cuda_io_fail(e, "csr1 upload");
    k_narrow<<<kGrid, kBlock, 0, s>>>(static_cast<const uint64_t*>(ring.dev[slot]), n, d_dst + done,
                                      d_overflow);
    note_launch();
    if ((e = cudaGetLastError())) return cuda_io_fail(e, "k_narrow");
    if ((e = ring.release(slot, s))) return cuda_io_fail(e, "csr1 ring");
    done += n;
  }
  return GSPMM_OK;
}

int validate_indptr_host(const std::vector<uint32_t>& indptr, uint64_t m, std::string* why) {
  if (indptr[0] != 0) {
    *why = "indptr[0] != 0";
    return 1;
  }
  for (size_t r = 0; r + 1 < indptr.size(); ++r)
    if (indptr[r] > indptr[r + 1]) {
      *why = "indptr not monotone at row " + std::to_string(r + 1);
      return 1;
    }
  if (indptr.back() != m) {
    *why = "indices/edge_ids length != indptr[num_rows] = " + std::to_string(indptr.back());
    return 1;
  }
  return 0;
}

}  // namespace

// validate() (csr.cpp:111-156) of a device CSR whose indptr already passed
// the host checks; `why` receives the reference's message on failure.
// Returns a CUDA error, *bad = 1 when a rule is broken.
cudaError_t validate_csr_device(uint32_t rows, uint32_t cols, uint64_t m,
                                const std::vector<uint32_t>& h_indptr, const uint32_t* d_indptr,
                                const uint32_t* d_indices, const uint32_t* d_eids, cudaStream_t s,
                                int* bad, std::string* why) {
  *bad = 0;
  if (m == 0) return cudaSuccess;
  unsigned long long* d_bad = nullptr;  // [0] range, [1] permutation, [2] order
  uint32_t* d_first = nullptr;
  uint32_t* d_bits = nullptr;
  const size_t bit_words = (m >> 5) + 1;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d_bad), 3 * sizeof(unsigned long long), s);
  if (!e) e = cudaMallocAsync(reinterpret_cast<void**>(&d_first), m * sizeof(uint32_t), s);
  if (!e) e = cudaMallocAsync(reinterpret_cast<void**>(&d_bits), bit_words * sizeof(uint32_t), s);
  if (!e) e = cudaMemsetAsync(d_bad, 0xff, 3 * sizeof(unsigned long long), s);
  if (!e) e = cudaMemsetAsync(d_first, 0xff, m * sizeof(uint32_t), s);
  if (!e) e = cudaMemsetAsync(d_bits, 0, bit_words * sizeof(uint32_t), s);
  unsigned long long h_bad[3] = {~0ull, ~0ull, ~0ull};
  if (!e) {
    k_check_range<<<kGrid, kBlock, 0, s>>>(d_indices, m, cols, d_bad + 0);
    k_first_use<<<kGrid, kBlock, 0, s>>>(d_eids, m, d_first);
    k_check_perm<<<kGrid, kBlock, 0, s>>>(d_eids, m, d_first, d_bad + 1);
    k_mark_row_starts<<<kGrid, kBlock, 0, s>>>(d_indptr, rows, m, d_bits);
    k_check_sorted<<<kGrid, kBlock, 0, s>>>(d_indices, d_eids, m, d_bits, d_bad + 2);
    note_launch(5);
    e = cudaGetLastError();
  }
  if (!e) e = cudaMemcpyAsync(h_bad, d_bad, sizeof(h_bad), cudaMemcpyDeviceToHost, s);
  if (d_bad) cudaFreeAsync(d_bad, s);
  if (d_first) cudaFreeAsync(d_first, s);
  if (d_bits) cudaFreeAsync(d_bits, s);
  if (!e) e = cudaStreamSynchronize(s);
  if (e) return e;
  // the reference's rule order: range, permutation, row order
  if (h_bad[0] != ~0ull) {
    *why = "index out of range at nonzero " + std::to_string(h_bad[0]);
  } else if (h_bad[1] != ~0ull) {
    *why = "edge_ids not a permutation (at nonzero " + std::to_string(h_bad[1]) + ")";
  } else if (h_bad[2] != ~0ull) {
    // the row holding nonzero h_bad[2] - 1: last row with indptr[r] <= it
    const uint64_t j = h_bad[2] - 1;
    const size_t r = std::upper_bound(h_indptr.begin(), h_indptr.end(), static_cast<uint32_t>(j)) -
                     h_indptr.begin() - 1;
    *why = "row " + std::to_string(r) + " not sorted at nonzero " + std::to_string(h_bad[2]);
  } else {
    return cudaSuccess;
  }
  *bad = 1;
  return cudaSuccess;
}

}  // namespace gspmm_b200

using namespace gspmm_b200;

extern "C" {

// ---- FMAT1 (io.cpp:137-166) -------------------------------------------------

int gspmm_fmat1_info(const char* path, int64_t* rows, int64_t* dim) {
  if (!path || !rows || !dim) return set_last_error(GSPMM_ERR_ARG, "null argument");
  InFile in(path);
  Fmat1Header h;
  const int st = read_fmat1_header(in, &h);
  if (st) return st;
  *rows = h.rows;
  *dim = h.dim;
  return GSPMM_OK;
}

int gspmm_fmat1_read(const char* path, float* data, int64_t ld) {
  if (!path) return set_last_error(GSPMM_ERR_ARG, "null argument");
  InFile in(path);
  Fmat1Header h;
  const int st = read_fmat1_header(in, &h);
  if (st) return st;
  if (h.rows * h.dim == 0) return GSPMM_OK;
  if (!data) return set_last_error(GSPMM_ERR_ARG, "null argument");
  if (ld == 0) ld = h.dim;
  if (ld < h.dim) return set_last_error(GSPMM_ERR_ARG, "ld smaller than the matrix width");
  if (ld == h.dim) {
    if (!in.read(data, static_cast<size_t>(h.rows * h.dim) * 4, Fmat1Header::kBytes))
      return io_fail(in.path + ": truncated data section");
    return GSPMM_OK;
  }
  for (int64_t r = 0; r < h.rows; ++r)
    if (!in.read(data + r * ld, static_cast<size_t>(h.dim) * 4,
                 Fmat1Header::kBytes + static_cast<uint64_t>(r * h.dim) * 4))
      return io_fail(in.path + ": truncated data section");
  return GSPMM_OK;
}

int gspmm_fmat1_read_device(const char* path, int device, float* d_data, int64_t ld, void* stream) {
  if (!path) return set_last_error(GSPMM_ERR_ARG, "null argument");
  InFile in(path);
  Fmat1Header h;
  const int st = read_fmat1_header(in, &h);
  if (st) return st;
  if (h.rows * h.dim == 0) return GSPMM_OK;
  if (!d_data) return set_last_error(GSPMM_ERR_ARG, "null argument");
  if (ld == 0) ld = h.dim;
  if (ld < h.dim) return set_last_error(GSPMM_ERR_ARG, "ld smaller than the matrix width");
  cudaError_t e = cudaSetDevice(device);
  if (e) return cuda_io_fail(e, "cudaSetDevice");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Ring ring;
  if ((e = ring.init(false))) return cuda_io_fail(e, "fmat1 ring");
  const uint64_t row_bytes = static_cast<uint64_t>(h.dim) * 4;
  if (row_bytes > kChunkBytes) return set_last_error(GSPMM_ERR_ARG, "matrix row wider than the staging ring");
  const int64_t per = static_cast<int64_t>(kChunkBytes / row_bytes);
  int slot = 0;
  for (int64_t r0 = 0; r0 < h.rows; slot ^= 1) {
    const int64_t n = std::min<int64_t>(per, h.rows - r0);
    if ((e = ring.acquire(slot))) return cuda_io_fail(e, "fmat1 ring");
    if (!in.read(ring.host[slot], static_cast<size_t>(n) * row_bytes,
                 Fmat1Header::kBytes + static_cast<uint64_t>(r0) * row_bytes))
      return io_fail(in.path + ": truncated data section");
    if ((e = cudaMemcpy2DAsync(d_data + r0 * ld, static_cast<size_t>(ld) * 4, ring.host[slot], row_bytes,
                               row_bytes, static_cast<size_t>(n), cudaMemcpyHostToDevice, s)))
      return cuda_io_fail(e, "fmat1 upload");
    if ((e = ring.release(slot, s))) return cuda_io_fail(e, "fmat1 ring");
    r0 += n;
  }
  if ((e = cudaStreamSynchronize(s))) return cuda_io_fail(e, "fmat1 upload");
  return GSPMM_OK;
}

int gspmm_fmat1_write(const char* path, const float* data, int64_t rows, int64_t dim, int64_t ld) {
  if (!path || rows < 0 || dim < 0 || (rows * dim && !data))
    return set_last_error(GSPMM_ERR_ARG, "null or negative argument");
  if (ld == 0) ld = dim;
  OutFile out(path);
  if (!out.f) return io_fail("cannot open " + out.path + " for writing");
  const uint64_t hdr[2] = {static_cast<uint64_t>(rows), static_cast<uint64_t>(dim)};
  bool ok = out.write("FMAT1", 5) && out.write(hdr, 16);
  if (ld == dim) {
    ok = ok && out.write(data, static_cast<size_t>(rows * dim) * 4);
  } else {
    for (int64_t r = 0; ok && r < rows; ++r) ok = out.write(data + r * ld, static_cast<size_t>(dim) * 4);
  }
  ok = out.close() && ok;
  return ok ? GSPMM_OK : io_fail("write failed: " + out.path);
}

// ---- CSR1 (io.cpp:168-205) --------------------------------------------------

int gspmm_csr1_info(const char* path, int* orientation, uint64_t* num_rows, uint64_t* num_cols,
                    uint64_t* num_edges) {
  if (!path) return set_last_error(GSPMM_ERR_ARG, "null argument");
  InFile in(path);
  Csr1Header h;
  const int st = read_csr1_header(in, &h);
  if (st) return st;
  if (orientation) *orientation = h.orientation;
  if (num_rows) *num_rows = h.rows;
  if (num_cols) *num_cols = h.cols;
  if (num_edges) *num_edges = h.edges;
  return GSPMM_OK;
}

int gspmm_csr1_read(const char* path, uint32_t* indptr, uint32_t* indices, uint32_t* edge_ids) {
  if (!path || !indptr) return set_last_error(GSPMM_ERR_ARG, "null argument");
  InFile in(path);
  Csr1Header h;
  int st = read_csr1_header(in, &h);
  if (st) return st;
  if (h.edges && (!indices || !edge_ids)) return set_last_error(GSPMM_ERR_ARG, "null argument");
  if ((st = read_u64_as_u32(in, h.indptr_off(), h.rows + 1, indptr))) return st;
  if ((st = read_u64_as_u32(in, h.indices_off(), h.edges, indices))) return st;
  if ((st = read_u64_as_u32(in, h.eids_off(), h.edges, edge_ids))) return st;
  // validate() on the payload (io.cpp:201-203)
  std::string why;
  const std::vector<uint32_t> ip(indptr, indptr + h.rows + 1);
  if (validate_indptr_host(ip, h.edges, &why)) return io_fail(in.path + ": invalid CSR payload: " + why);
  st = validate_csr_host(static_cast<uint32_t>(h.rows), static_cast<uint32_t>(h.cols), indptr, indices,
                         edge_ids);
  if (st) return io_fail(in.path + ": invalid CSR payload: " + gspmm_last_error());
  return GSPMM_OK;
}

int gspmm_csr1_write(const char* path, int orientation, uint32_t num_rows, uint32_t num_cols,
                     const uint32_t* indptr, const uint32_t* indices, const uint32_t* edge_ids) {
  if (!path || !indptr) return set_last_error(GSPMM_ERR_ARG, "null argument");
  const uint64_t m = indptr[num_rows];
  if (m && (!indices || !edge_ids)) return set_last_error(GSPMM_ERR_ARG, "null argument");
  OutFile out(path);
  if (!out.f) return io_fail("cannot open " + out.path + " for writing");
  const char orient = orientation == GSPMM_DST_MAJOR ? 1 : 0;
  const uint64_t hdr[3] = {num_rows, num_cols, m};
  bool ok = out.write("CSR1", 4) && out.write(&orient, 1) && out.write(hdr, 24);
  std::vector<uint64_t> buf(1u << 16);
  auto widen = [&](const uint32_t* a, uint64_t count) {
    for (uint64_t done = 0; ok && done < count;) {
      const uint64_t n = std::min<uint64_t>(buf.size(), count - done);
      for (uint64_t i = 0; i < n; ++i) buf[i] = a[done + i];
      ok = out.write(buf.data(), n * 8);
      done += n;
    }
  };
  widen(indptr, static_cast<uint64_t>(num_rows) + 1);
  widen(indices, m);
  widen(edge_ids, m);
  ok = out.close() && ok;
  return ok ? GSPMM_OK : io_fail("write failed: " + out.path);
}

int gspmm_graph_load_csr1(const char* path, int device, gspmm_graph* out) {
  if (!path || !out) return set_last_error(GSPMM_ERR_ARG, "null argument");
  InFile in(path);
  Csr1Header h;
  int st = read_csr1_header(in, &h);
  if (st) return st;
  // indptr: small, narrowed and checked on the host (it also feeds the plan)
  std::vector<uint32_t> indptr(h.rows + 1);
  if ((st = read_u64_as_u32(in, h.indptr_off(), h.rows + 1, indptr.data()))) return st;
  std::string why;
  if (validate_indptr_host(indptr, h.edges, &why))
    return io_fail(in.path + ": invalid CSR payload: " + why);

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_last_error(GSPMM_ERR_CUDA, "no CUDA device visible: the B200 kernels cannot run here");
  if (device < 0 || device >= ndev) return set_last_error(GSPMM_ERR_ARG, "device index out of range");
  cudaError_t e = cudaSetDevice(device);
  if (e) return cuda_io_fail(e, "cudaSetDevice");
  cudaStream_t s = nullptr;
  if ((e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking))) return cuda_io_fail(e, "csr1 stream");
  uint32_t *d_indptr = nullptr, *d_indices = nullptr, *d_eids = nullptr, *d_overflow = nullptr;
  auto done = [&](int status) {
    cudaStreamSynchronize(s);
    cudaFree(d_indptr);
    cudaFree(d_indices);
    cudaFree(d_eids);
    cudaFree(d_overflow);
    cudaStreamDestroy(s);
    return status;
  };
  const uint64_t m = h.edges;
  if ((e = cudaMalloc(&d_indptr, 4 * (h.rows + 1))) || (e = cudaMalloc(&d_indices, 4 * std::max<uint64_t>(m, 1))) ||
      (e = cudaMalloc(&d_eids, 4 * std::max<uint64_t>(m, 1))) || (e = cudaMalloc(&d_overflow, 4)) ||
      (e = cudaMemsetAsync(d_overflow, 0, 4, s)) ||
      (e = cudaMemcpyAsync(d_indptr, indptr.data(), 4 * (h.rows + 1), cudaMemcpyHostToDevice, s)))
    return done(cuda_io_fail(e, "csr1 device arrays"));
  {
    Ring ring;
    if ((e = ring.init(true))) return done(cuda_io_fail(e, "csr1 ring"));
    if ((st = stream_u64_to_device(in, h.indices_off(), m, d_indices, ring, d_overflow, s))) return done(st);
    if ((st = stream_u64_to_device(in, h.eids_off(), m, d_eids, ring, d_overflow, s))) return done(st);
    uint32_t overflow = 0;
    if ((e = cudaMemcpyAsync(&overflow, d_overflow, 4, cudaMemcpyDeviceToHost, s)) ||
        (e = cudaStreamSynchronize(s)))
      return done(cuda_io_fail(e, "csr1 upload"));
    if (overflow) return done(io_fail(in.path + ": id does not fit the configured id width"));
  }
  int bad = 0;
  if ((e = validate_csr_device(static_cast<uint32_t>(h.rows), static_cast<uint32_t>(h.cols), m, indptr,
                               d_indptr, d_indices, d_eids, s, &bad, &why)))
    return done(cuda_io_fail(e, "csr1 validate"));
  if (bad) return done(io_fail(in.path + ": invalid CSR payload: " + why));
  st = gspmm_graph_create_device(device, h.orientation, static_cast<uint32_t>(h.rows),
                                 static_cast<uint32_t>(h.cols), d_indptr, d_indices, d_eids, out);
  return done(st);
}

int gspmm_validate_csr_device(int device, uint32_t num_rows, uint32_t num_cols, const uint32_t* d_indptr,
                              const uint32_t* d_indices, const uint32_t* d_edge_ids, void* stream) {
  if (!d_indptr) return set_last_error(GSPMM_ERR_ARG, "null argument");
  cudaError_t e = cudaSetDevice(device);
  if (e) return cuda_io_fail(e, "cudaSetDevice");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<uint32_t> indptr(static_cast<size_t>(num_rows) + 1);
  if ((e = cudaMemcpyAsync(indptr.data(), d_indptr, 4 * indptr.size(), cudaMemcpyDeviceToHost, s)) ||
      (e = cudaStreamSynchronize(s)))
    return cuda_io_fail(e, "download indptr");
  std::string why;
  if (indptr[0] != 0) return set_last_error(GSPMM_ERR_STRUCTURE, "indptr[0] != 0");
  for (uint32_t r = 0; r < num_rows; ++r)
    if (indptr[r] > indptr[r + 1])
      return set_last_error(GSPMM_ERR_STRUCTURE, "indptr not monotone at row " + std::to_string(r + 1));
  const uint64_t m = indptr[num_rows];
  if (m && (!d_indices || !d_edge_ids)) return set_last_error(GSPMM_ERR_ARG, "null CSR array");
  int bad = 0;
  if ((e = validate_csr_device(num_rows, num_cols, m, indptr, d_indptr, d_indices, d_edge_ids, s, &bad, &why)))
    return cuda_io_fail(e, "validate_csr_device");
  return bad ? set_last_error(GSPMM_ERR_STRUCTURE, why) : GSPMM_OK;
}

// ---- text edge lists (io.cpp:80-135) ---------------------------------------

namespace {
bool parse_field(const char*& s, const char* end, uint64_t& out) {
  while (s < end && (*s == ' ' || *s == '\t')) ++s;
  const auto [ptr, ec] = std::from_chars(s, end, out);
  if (ec != std::errc{} || ptr == s) return false;
  s = ptr;
  while (s < end && (*s == ' ' || *s == '\t')) ++s;
  return true;
}
}  // namespace

int gspmm_edge_list_read(const char* path, uint32_t* num_nodes, uint64_t* num_edges, uint32_t** src,
                         uint32_t** dst) {
  if (!path || !num_nodes || !num_edges || !src || !dst)
    return set_last_error(GSPMM_ERR_ARG, "null argument");
  InFile in(path);
  if (!in.ok()) return io_fail("cannot open " + in.path);
  std::vector<char> text(in.size);
  if (in.size && !in.read(text.data(), in.size, 0)) return io_fail("cannot open " + in.path);
  std::vector<uint32_t> s_ids, d_ids;
  bool have_header = false;
  uint64_t header_nodes = 0, max_id = 0, lineno = 0;
  constexpr uint64_t id_cap = std::numeric_limits<uint32_t>::max();
  auto line_error = [&](const char* what) {
    return set_last_error(GSPMM_ERR_PARSE, in.path + ":" + std::to_string(lineno) + ": " + what);
  };
  const char* p = text.data();
  const char* const file_end = p + text.size();
  while (p < file_end) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(file_end - p)));
    const char* line_end = nl ? nl : file_end;
    ++lineno;
    const char* hash = static_cast<const char*>(std::memchr(p, '#', static_cast<size_t>(line_end - p)));
    const char* end = hash ? hash : line_end;
    const char* s = p;
    p = nl ? nl + 1 : file_end;
    while (s < end && (*s == ' ' || *s == '\t' || *s == '\r')) ++s;
    if (s == end) continue;
    if (*s == '%') {
      if (std::string_view(s, static_cast<size_t>(end - s)).rfind("%nodes", 0) != 0)
        return line_error("unknown '%' directive");
      const char* q = s + 6;
      uint64_t n = 0;
      if (!parse_field(q, end, n)) return line_error("bad %nodes value");
      if (n > id_cap) return line_error("%nodes overflows id width");
      have_header = true;
      header_nodes = n;
      continue;
    }
    uint64_t a = 0, b = 0;
    if (!parse_field(s, end, a) || !parse_field(s, end, b)) return line_error("expected 'src dst'");
    while (s < end && *s == '\r') ++s;
    if (s != end) return line_error("trailing garbage after edge");
    if (a >= id_cap || b >= id_cap) return line_error("node id overflows id width");
    if (have_header && (a >= header_nodes || b >= header_nodes)) return line_error("node id >= %nodes");
    max_id = std::max({max_id, a, b});
    s_ids.push_back(static_cast<uint32_t>(a));
    d_ids.push_back(static_cast<uint32_t>(b));
  }
  const size_t m = s_ids.size();
  *num_nodes = have_header ? static_cast<uint32_t>(header_nodes) : m == 0 ? 0u : static_cast<uint32_t>(max_id + 1);
  *num_edges = m;
  *src = static_cast<uint32_t*>(std::malloc(std::max<size_t>(m, 1) * 4));
  *dst = static_cast<uint32_t*>(std::malloc(std::max<size_t>(m, 1) * 4));
  if (!*src || !*dst) {
    std::free(*src);
    std::free(*dst);
    *src = *dst = nullptr;
    return io_fail(in.path + ": out of memory");
  }
  if (m) {
    std::memcpy(*src, s_ids.data(), m * 4);
    std::memcpy(*dst, d_ids.data(), m * 4);
  }
  return GSPMM_OK;
}

int gspmm_edge_list_write(const char* path, uint32_t num_nodes, uint64_t num_edges, const uint32_t* src,
                          const uint32_t* dst) {
  if (!path || (num_edges && (!src || !dst))) return set_last_error(GSPMM_ERR_ARG, "null argument");
  OutFile out(path);
  if (!out.f) return io_fail("cannot open " + out.path + " for writing");
  bool ok = std::fprintf(out.f, "%%nodes %u\n", num_nodes) > 0;
  for (uint64_t i = 0; ok && i < num_edges; ++i) ok = std::fprintf(out.f, "%u %u\n", src[i], dst[i]) > 0;
  ok = out.close() && ok;
  return ok ? GSPMM_OK : io_fail("write failed: " + out.path);
}

}  // extern "C"
