"""Generates the container fixtures tests/golden/io_*.{csr,fmat,txt} with the
UNMODIFIED reference library's own writers (save_csr / save_feature_matrix /
save_edge_list, io.cpp:129-181, through oracle/_ref).  Run where
/root/reference exists:  python tests/golden/make_golden_io.py

The graphs are test_util.hpp's random_small_graph(1) and (8) (the seeds of
test_io.cpp:104), both orientations; the matrix is random_features(37, 5, 123)
(test_io.cpp:93)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
sys.path.insert(0, HERE)
from oracle import oracle as O  # noqa: E402
from make_golden import small_graph_via_ref  # noqa: E402

assert O.ref_available(), "oracle/_ref/libgspmm_ref.so missing: run make -C oracle"

meta = {}
for seed in (1, 8):
    n, src, dst = small_graph_via_ref(seed)
    O.ref_save_edge_list(os.path.join(HERE, f"io_graph{seed}.txt"), n, src, dst)
    for orient, tag in ((O.SRC_MAJOR, "src"), (O.DST_MAJOR, "dst")):
        csr = O.ref_build_csr(n, src, dst, orient)
        O.ref_save_csr(os.path.join(HERE, f"io_graph{seed}_{tag}.csr"), orient, n, n, *csr)
        for k, a in zip(("indptr", "indices", "eids"), csr):
            meta[f"g{seed}_{tag}_{k}"] = a
    meta[f"g{seed}_n"] = np.array([n])
    meta[f"g{seed}_src"], meta[f"g{seed}_dst"] = src, dst
x = O.ref_random_features(37, 5, 123)
O.ref_save_feature_matrix(os.path.join(HERE, "io_feats.fmat"), x)
meta["feats"] = x
np.savez_compressed(os.path.join(HERE, "io_expected.npz"), **meta)
print(sorted(f for f in os.listdir(HERE) if f.startswith("io_")))
