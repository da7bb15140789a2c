// synth.cpp -- input synthesis and canonical CSR construction on the host.
//
// These produce the benchmark/test inputs the reference builds with its own
// generators (generate.cpp) and CSR builder (csr.cpp), bit for bit, but in
// parallel so the 17M-124M edge configs build in seconds:
//   * R-MAT: the reference draws edges sequentially from one counter stream,
//     each TRY consuming `levels` consecutive counters and rejected tries
//     (u or v >= n) simply being skipped (generate.cpp:140-172).  Try i
//     therefore always reads counters [i*levels, (i+1)*levels): tries are
//     evaluated in parallel and the first num_edges accepted ones, in try
//     order, are the reference's edges.
//   * canonical CSR (csr.cpp:31-71: rows ascending, then neighbour, then
//     edge id) is built as a parallel row histogram + scatter followed by a
//     per-row sort on the (neighbour, edge id) key -- the same total order
//     as the reference's two stable counting sorts.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <thread>
#include <vector>

#include "gspmm_b200.h"

namespace {

int resolve_threads(int threads) {
  if (threads > 0) return threads;
  const unsigned hc = std::thread::hardware_concurrency();
  return hc ? static_cast<int>(std::min(hc, 128u)) : 1;
}

// Static partition of [0, n) over T threads.
void parallel_for(int64_t n, int threads, const std::function<void(int64_t, int64_t, int)>& fn) {
  const int T = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(resolve_threads(threads), n)));
  if (T == 1) {
    fn(0, n, 0);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(T);
  for (int t = 0; t < T; ++t) {
    const int64_t b = n * t / T, e = n * (t + 1) / T;
    pool.emplace_back(fn, b, e, t);
  }
  for (auto& th : pool) th.join();
}

// Dynamic chunks for skewed per-row work.
void parallel_chunks(int64_t n, int64_t chunk, int threads,
                     const std::function<void(int64_t, int64_t)>& fn) {
  const int T = resolve_threads(threads);
  std::atomic<int64_t> next{0};
  auto worker = [&]() {
    for (;;) {
      const int64_t b = next.fetch_add(chunk);
      if (b >= n) return;
      fn(b, std::min(n, b + chunk));
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < T; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
}

inline uint64_t splitmix64_at(uint64_t seed, uint64_t counter) {
  uint64_t z = seed + (counter + 1) * 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline double u01_at(uint64_t seed, uint64_t counter) {
  return static_cast<double>(splitmix64_at(seed, counter) >> 11) * 0x1.0p-53;
}

struct RmatParams {
  uint32_t n;
  int levels;
  double a, t_ab, t_abc;
  uint64_t seed;
};

// One R-MAT try (the body of generate.cpp:159-167).
inline bool rmat_try(const RmatParams& P, uint64_t i, uint32_t& u, uint32_t& v) {
  u = 0;
  v = 0;
  const uint64_t c0 = i * static_cast<uint64_t>(P.levels);
  for (int l = 0; l < P.levels; ++l) {
    const double r = u01_at(P.seed, c0 + l);
    const int quad = r < P.a ? 0 : r < P.t_ab ? 1 : r < P.t_abc ? 2 : 3;
    u = (u << 1) | static_cast<uint32_t>(quad >> 1);
    v = (v << 1) | static_cast<uint32_t>(quad & 1);
  }
  return u < P.n && v < P.n;
}

}  // namespace

extern "C" {

void gspmm_free(void* p) { std::free(p); }

int64_t gspmm_synth_rmat(uint32_t n, uint64_t num_edges, double a, double b,
                         double c, double d, uint64_t seed, uint32_t* src,
                         uint32_t* dst, int threads) {
  (void)d;
  if (num_edges == 0) return 0;
  if (n == 0) return -GSPMM_ERR_CONFIG;
  RmatParams P;
  P.n = n;
  P.levels = 0;
  while ((uint64_t{1} << P.levels) < static_cast<uint64_t>(n)) ++P.levels;
  P.a = a;
  P.t_ab = a + b;
  P.t_abc = P.t_ab + c;
  P.seed = seed;
  const int T = resolve_threads(threads);
  uint64_t produced = 0, try0 = 0;
  int64_t run = 0;  // consecutive rejections carried across rounds
  while (produced < num_edges) {
    // Enough tries for the remaining edges with a small margin.
    const uint64_t need = num_edges - produced;
    const uint64_t tries = need + need / 8 + 1024;
    const uint64_t chunk = (tries + T - 1) / T;
    std::vector<uint64_t> acc(T, 0);
    std::vector<int64_t> lead(T, 0), maxrun(T, 0), tail(T, 0);
    parallel_for(T, T, [&](int64_t tb, int64_t te, int) {
      for (int64_t t = tb; t < te; ++t) {
        const uint64_t b = try0 + t * chunk, e = std::min(try0 + tries, b + chunk);
        uint64_t cnt = 0;
        int64_t r = 0, mr = 0, ld = -1;
        for (uint64_t i = b; i < e; ++i) {
          uint32_t u, v;
          if (rmat_try(P, i, u, v)) {
            if (ld < 0) ld = r;
            mr = std::max(mr, r);
            r = 0;
            ++cnt;
          } else {
            ++r;
          }
        }
        acc[t] = cnt;
        lead[t] = ld < 0 ? r : ld;
        maxrun[t] = ld < 0 ? -1 : mr;  // -1: no accept in this chunk
        tail[t] = r;
      }
    });
    // Reference fails an edge after more than 10000 rejected tries.
    for (int t = 0; t < T; ++t) {
      if (maxrun[t] < 0) {
        run += lead[t];
      } else {
        if (run + lead[t] > 10000 || maxrun[t] > 10000) return -GSPMM_ERR_CONFIG;
        run = tail[t];
      }
    }
    if (run > 10000) return -GSPMM_ERR_CONFIG;
    std::vector<uint64_t> off(T + 1, 0);
    for (int t = 0; t < T; ++t) off[t + 1] = off[t] + acc[t];
    parallel_for(T, T, [&](int64_t tb, int64_t te, int) {
      for (int64_t t = tb; t < te; ++t) {
        uint64_t pos = produced + off[t];
        if (pos >= num_edges) continue;
        const uint64_t b = try0 + t * chunk, e = std::min(try0 + tries, b + chunk);
        for (uint64_t i = b; i < e && pos < num_edges; ++i) {
          uint32_t u, v;
          if (rmat_try(P, i, u, v)) {
            src[pos] = u;
            dst[pos] = v;
            ++pos;
          }
        }
      }
    });
    produced = std::min<uint64_t>(num_edges, produced + off[T]);
    try0 += tries;
  }
  return static_cast<int64_t>(num_edges);
}

// Erdos-Renyi (generate.cpp:31-108): geometric skipping over the n*n cells
// with an exactly-searched table of (1-p)^k; sequential (one stream).
int64_t gspmm_synth_er(uint32_t n, uint64_t num_edges, double prob, uint64_t seed,
                       uint32_t** src, uint32_t** dst) {
  double p = prob;
  if (p < 0.0) {
    const double pairs = static_cast<double>(n) * (static_cast<double>(n) - 1.0);
    p = pairs > 0.0 ? static_cast<double>(num_edges) / pairs : 0.0;
  }
  std::vector<uint32_t> s, t;
  const uint64_t cells = static_cast<uint64_t>(n) * n;
  uint64_t counter = 0;
  auto emit = [&](uint64_t cell) {
    const uint32_t i = static_cast<uint32_t>(cell / n), j = static_cast<uint32_t>(cell % n);
    if (i != j) {
      s.push_back(i);
      t.push_back(j);
    }
  };
  if (p > 0.0 && cells > 0) {
    if (p >= 1.0) {
      for (uint64_t c = 0; c < cells; ++c) emit(c);
    } else {
      std::vector<double> pow_q{1.0};
      const double q = 1.0 - p;
      double x = q;
      while (x > 0x1.0p-64 && pow_q.size() < 4096) {
        pow_q.push_back(x);
        x *= q;
      }
      pow_q.push_back(x);
      auto gap = [&](double uu) -> uint64_t {
        double tt = 1.0 - uu;
        const size_t last = pow_q.size() - 1;
        uint64_t base = 0;
        while (tt <= pow_q[last]) {
          base += last;
          tt /= pow_q[last];
        }
        size_t lo = 1, hi = last;
        while (lo < hi) {
          const size_t mid = (lo + hi) / 2;
          if (pow_q[mid] < tt) hi = mid; else lo = mid + 1;
        }
        return base + lo - 1;
      };
      uint64_t pos = gap(u01_at(seed, counter++));
      while (pos < cells) {
        emit(pos);
        pos += 1 + gap(u01_at(seed, counter++));
      }
    }
  }
  const size_t m = s.size();
  *src = static_cast<uint32_t*>(std::malloc(std::max<size_t>(m, 1) * sizeof(uint32_t)));
  *dst = static_cast<uint32_t*>(std::malloc(std::max<size_t>(m, 1) * sizeof(uint32_t)));
  if (m) {
    std::memcpy(*src, s.data(), m * sizeof(uint32_t));
    std::memcpy(*dst, t.data(), m * sizeof(uint32_t));
  }
  return static_cast<int64_t>(m);
}

}  // extern "C"

namespace {
// Canonical CSR from (row, col, eid) triples given implicitly by accessors.
template <class RowOf, class ColOf, class EidOf>
void canonical_csr(uint32_t num_rows, int64_t m, RowOf row_of, ColOf col_of, EidOf eid_of,
                   uint32_t* indptr, uint32_t* indices, uint32_t* eids, int threads) {
  std::vector<std::atomic<uint32_t>> cnt(static_cast<size_t>(num_rows) + 1);
  parallel_for(static_cast<int64_t>(num_rows) + 1, threads, [&](int64_t b, int64_t e, int) {
    for (int64_t i = b; i < e; ++i) cnt[i].store(0, std::memory_order_relaxed);
  });
  parallel_for(m, threads, [&](int64_t b, int64_t e, int) {
    for (int64_t i = b; i < e; ++i) cnt[row_of(i)].fetch_add(1, std::memory_order_relaxed);
  });
  indptr[0] = 0;
  for (uint32_t r = 0; r < num_rows; ++r)
    indptr[r + 1] = indptr[r] + cnt[r].load(std::memory_order_relaxed);
  parallel_for(num_rows, threads, [&](int64_t b, int64_t e, int) {
    for (int64_t r = b; r < e; ++r) cnt[r].store(indptr[r], std::memory_order_relaxed);
  });
  std::vector<uint64_t> key(static_cast<size_t>(std::max<int64_t>(m, 1)));
  parallel_for(m, threads, [&](int64_t b, int64_t e, int) {
    for (int64_t i = b; i < e; ++i) {
      const uint32_t pos = cnt[row_of(i)].fetch_add(1, std::memory_order_relaxed);
      key[pos] = (static_cast<uint64_t>(col_of(i)) << 32) | eid_of(i);
    }
  });
  parallel_chunks(num_rows, 4096, threads, [&](int64_t b, int64_t e) {
    for (int64_t r = b; r < e; ++r) {
      std::sort(key.begin() + indptr[r], key.begin() + indptr[r + 1]);
      for (uint32_t j = indptr[r]; j < indptr[r + 1]; ++j) {
        indices[j] = static_cast<uint32_t>(key[j] >> 32);
        eids[j] = static_cast<uint32_t>(key[j]);
      }
    }
  });
}
}  // namespace

extern "C" {

int gspmm_build_csr(uint32_t n, int64_t m, const uint32_t* src, const uint32_t* dst,
                    int orientation, uint32_t* indptr, uint32_t* indices,
                    uint32_t* edge_ids, int threads) {
  for (int64_t i = 0; i < m; ++i)
    if (src[i] >= n || dst[i] >= n) return GSPMM_ERR_STRUCTURE;
  const bool dm = orientation == GSPMM_DST_MAJOR;
  canonical_csr(
      n, m, [&](int64_t i) { return dm ? dst[i] : src[i]; },
      [&](int64_t i) { return dm ? src[i] : dst[i]; },
      [](int64_t i) { return static_cast<uint32_t>(i); }, indptr, indices, edge_ids, threads);
  return GSPMM_OK;
}

int gspmm_transpose(uint32_t num_rows, uint32_t num_cols, const uint32_t* indptr,
                    const uint32_t* indices, const uint32_t* edge_ids, uint32_t* t_indptr,
                    uint32_t* t_indices, uint32_t* t_edge_ids, int threads) {
  const int64_t m = indptr[num_rows];
  std::vector<uint32_t> row(static_cast<size_t>(std::max<int64_t>(m, 1)));
  parallel_chunks(num_rows, 4096, threads, [&](int64_t b, int64_t e) {
    for (int64_t r = b; r < e; ++r)
      for (uint32_t j = indptr[r]; j < indptr[r + 1]; ++j) row[j] = static_cast<uint32_t>(r);
  });
  canonical_csr(
      num_cols, m, [&](int64_t j) { return indices[j]; }, [&](int64_t j) { return row[j]; },
      [&](int64_t j) { return edge_ids[j]; }, t_indptr, t_indices, t_edge_ids, threads);
  return GSPMM_OK;
}

void gspmm_synth_uniform(int64_t count, uint64_t seed, float* out, int threads) {
  parallel_for(count, threads, [&](int64_t b, int64_t e, int) {
    for (int64_t i = b; i < e; ++i) {
      const float u = static_cast<float>(splitmix64_at(seed, static_cast<uint64_t>(i)) >> 40) *
                      0x1.0p-24f;
      out[i] = 2.0f * u - 1.0f;
    }
  });
}

// Box-Muller on u01 draws 2i, 2i+1 in double, rounded once.
void gspmm_synth_normal(int64_t count, uint64_t seed, float* out, int threads) {
  parallel_for(count, threads, [&](int64_t b, int64_t e, int) {
    for (int64_t i = b; i < e; ++i) {
      const double u1 = u01_at(seed, 2 * static_cast<uint64_t>(i));
      const double u2 = u01_at(seed, 2 * static_cast<uint64_t>(i) + 1);
      const double r = std::sqrt(-2.0 * std::log(1.0 - u1));
      out[i] = static_cast<float>(r * std::cos(6.283185307179586476925286766559 * u2));
    }
  });
}

int64_t gspmm_synth_powerlaw(uint32_t n, uint32_t d_min, uint32_t d_max, uint64_t seed,
                             uint32_t* src, uint32_t* dst, int threads) {
  if (n == 0 || d_min == 0 || d_max < d_min) return -GSPMM_ERR_CONFIG;
  // in-degree of node v: inverse CDF of P(d) ~ d^-2 on [d_min, d_max]
  const double a = 1.0 / d_min, b = 1.0 / d_min - 1.0 / d_max;
  std::vector<uint64_t> off(static_cast<size_t>(n) + 1, 0);
  parallel_for(n, threads, [&](int64_t lo, int64_t hi, int) {
    for (int64_t v = lo; v < hi; ++v) {
      const double u = u01_at(seed, static_cast<uint64_t>(v));
      double d = std::floor(1.0 / (a - u * b));
      if (d < d_min) d = d_min;
      if (d > d_max) d = d_max;
      off[v + 1] = static_cast<uint64_t>(d);
    }
  });
  for (uint32_t v = 0; v < n; ++v) off[v + 1] += off[v];
  const uint64_t m = off[n];
  if (!src || !dst) return static_cast<int64_t>(m);
  const uint64_t seed2 = seed ^ 0x5851f42d4c957f2dULL;
  parallel_chunks(n, 256, threads, [&](int64_t lo, int64_t hi) {
    for (int64_t v = lo; v < hi; ++v)
      for (uint64_t e = off[v]; e < off[v + 1]; ++e) {
        const unsigned __int128 x = static_cast<unsigned __int128>(splitmix64_at(seed2, e)) * n;
        src[e] = static_cast<uint32_t>(x >> 64);
        dst[e] = static_cast<uint32_t>(v);
      }
  });
  return static_cast<int64_t>(m);
}

void gspmm_synth_gcn_weights(uint32_t n, int64_t m, const uint32_t* src, const uint32_t* dst,
                             float* w, int threads) {
  std::vector<std::atomic<uint32_t>> dout(n), din(n);
  parallel_for(n, threads, [&](int64_t b, int64_t e, int) {
    for (int64_t i = b; i < e; ++i) {
      dout[i].store(0, std::memory_order_relaxed);
      din[i].store(0, std::memory_order_relaxed);
    }
  });
  parallel_for(m, threads, [&](int64_t b, int64_t e, int) {
    for (int64_t i = b; i < e; ++i) {
      dout[src[i]].fetch_add(1, std::memory_order_relaxed);
      din[dst[i]].fetch_add(1, std::memory_order_relaxed);
    }
  });
  parallel_for(m, threads, [&](int64_t b, int64_t e, int) {
    for (int64_t i = b; i < e; ++i) {
      const double a = static_cast<double>(dout[src[i]].load(std::memory_order_relaxed));
      const double c = static_cast<double>(din[dst[i]].load(std::memory_order_relaxed));
      w[i] = static_cast<float>(1.0 / std::sqrt(a * c));
    }
  });
}

}  // extern "C"
