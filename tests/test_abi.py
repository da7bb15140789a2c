"""CPU-only checks of the product boundary: the C-ABI library loads, exports
every symbol include/gspmm_b200.h declares, its descriptor helpers follow
the reference's rules, and the host-side input synthesis / CSR builder
reproduce the reference (via the pinned oracle) bit for bit."""
import os
import re

import numpy as np
import pytest

import paper_2007_06354_b200 as P
from paper_2007_06354_b200 import _capi as A
from oracle import oracle as O
from gspmm_testutil import HAS_GPU, ROOT


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "gspmm_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gspmm_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(A.LIB, s), s
        assert s in A.SIGNATURES, f"{s} has no ctypes prototype"


def test_abi_version():
    assert A.LIB.gspmm_abi_version() == 3


def test_plan_struct_mirrors_the_header():
    # gspmm_plan (include/gspmm_b200.h): the ctypes mirror has the header's
    # fields in the header's order (six 32-bit words)
    import ctypes
    import re
    hdr = open(os.path.join(ROOT, "include", "gspmm_b200.h")).read()
    body = hdr[:hdr.index("} gspmm_plan;")]
    body = body[body.rindex("typedef struct {"):]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"(?:uint32_t|int32_t)\s+(\w+)\s*;", body)
    assert fields == [f[0] for f in A.Plan._fields_]
    assert ctypes.sizeof(A.Plan) == 4 * len(fields) == 24


def test_library_path_is_in_tree():
    assert os.path.commonpath([P.LIB_PATH, ROOT]) == ROOT


ALL_NAMES = []
for lhs in "uve":
    for red in ("add", "max", "min", "mul", "copy"):
        ALL_NAMES.append(f"{lhs}_copy_{red}_v")
        for rhs in "uve":
            for binop in ("add", "sub", "mul", "div", "dot"):
                for out in "uve":
                    ALL_NAMES.append(f"{lhs}_{binop}_{rhs}_{red}_{out}")
ALL_NAMES += ["u_copy_add_u", "bogus", "u_mul", "u_copy_add_v_x", "u_foo_e_add_v",
              "v_copy_add_u", "u_copy_sum_v", ""]


@pytest.mark.parametrize("name", ALL_NAMES)
def test_named_config_matches_reference_grammar(name):  # br_config.cpp:96-131
    try:
        want = O.named_config(name)
    except O.OracleError:
        want = None
    if want is None:
        with pytest.raises(P.ConfigError):
            P.named_config(name)
    else:
        assert P.named_config(name).astuple() == want


def test_validate_config_rules():  # br_config.cpp:83-94
    P.validate_config((P.U, P.NONE, P.COPY, P.SUM, P.V))
    bad = [(P.NONE, P.NONE, P.COPY, P.SUM, P.V), (P.U, P.NONE, P.COPY, P.SUM, P.NONE),
           (P.U, P.E, P.COPY, P.SUM, P.V), (P.U, P.NONE, P.MUL, P.SUM, P.V),
           (P.U, P.U, P.MUL, P.SUM, P.V), (P.U, P.V, P.DOT, P.SUM, P.E)]
    for cfg in bad:
        with pytest.raises(P.ConfigError):
            P.validate_config(cfg)
    # constructed (not named) v_copy_add_u is accepted, as in the reference
    P.validate_config((P.V, P.NONE, P.COPY, P.SUM, P.U))


def test_required_orientation():  # kernels.cpp:400-411
    for s in (P.PULL, P.BLOCKED, P.SPMM):
        assert P.required_orientation(s, P.V) == P.DST_MAJOR
        assert P.required_orientation(s, P.E) == P.DST_MAJOR
        assert P.required_orientation(s, P.U) == P.SRC_MAJOR
    assert P.required_orientation(P.PUSH, P.V) == P.SRC_MAJOR
    with pytest.raises(P.ConfigError):
        P.required_orientation(P.SPMM, P.NONE)


@pytest.mark.parametrize("seed", range(4))
def test_synth_matches_oracle(seed):
    for (a, b, c, d) in ((0.57, 0.19, 0.19, 0.05), (0.40, 0.25, 0.25, 0.10)):
        for n in (1, 7, 1000, 1025):
            s, t = P.synth_rmat(n, 3000, a, b, c, d, seed, threads=1 + seed)
            s2, t2 = O.gen_rmat(n, 3000, a, b, c, d, seed)
            assert (s == s2).all() and (t == t2).all()
    s, t = P.synth_er(400, 3000, -1.0, seed)
    s2, t2 = O.gen_er(400, 3000, -1.0, seed)
    assert (s == s2).all() and (t == t2).all()
    s, t = O.gen_rmat(2000, 30000, seed=seed)
    for o in (P.SRC_MAJOR, P.DST_MAJOR):
        mine = P.build_csr(2000, s, t, o, threads=3)
        ref = O.build_csr(2000, s, t, o)
        assert all((x == y).all() for x, y in zip(mine, ref))
        tm = P.transpose(2000, 2000, *mine)
        tr = O.transpose(2000, 2000, *ref)
        assert all((x == y).all() for x, y in zip(tm, tr))
    assert (P.synth_uniform(77, 9, seed) == O.random_features(77, 9, seed)).all()
    assert (P.synth_normal(77, 9, seed) == O.normal_features(77, 9, seed)).all()
    assert (P.synth_gcn_weights(2000, s, t) == O.gcn_weights(2000, s, t)).all()


def test_powerlaw_generator_matches_oracle():
    for seed in range(3):
        s, d = P.synth_powerlaw(2000, 5, 400, seed, threads=3)
        s2, d2 = O.gen_powerlaw(2000, 5, 400, seed)
        assert (s == s2).all() and (d == d2).all()
        deg = np.bincount(d, minlength=2000)
        assert deg.min() >= 5 and deg.max() <= 400


def test_synth_empty_and_errors():
    s, t = P.synth_rmat(10, 0)
    assert len(s) == 0
    with pytest.raises(P.ConfigError):
        P.synth_rmat(0, 5)
    with pytest.raises(P.StructureError):
        P.build_csr(2, [0], [2])


@pytest.mark.skipif(HAS_GPU, reason="checks the no-device error path")
def test_no_device_fails_loudly():
    ip, ix, ei = O.build_csr(3, [0, 1], [2, 2])
    with pytest.raises(P.DeviceError):
        P.Graph(ip, ix, ei)


def test_graph_validation_runs_before_upload():
    # a malformed CSR is a StructureError even without a device
    with pytest.raises(P.StructureError):
        P.Graph(np.array([0, 2, 1], np.uint32), np.array([0], np.uint32),
                np.array([0], np.uint32), validate=True)
