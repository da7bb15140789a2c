"""One small pass through every kernel family, for compute-sanitizer
(scripts/gpu/sanitize.sh runs it under memcheck, racecheck, synccheck and
initcheck): k_gather (copy / mul / arith, sum / max+argmax / dual, source
blocks, VPL-5 wide units), k_long_rg (forced long rows: mbarrier ring,
cp.async id ring), k_rows, k_dot, k_dot_edges4, edge softmax fwd/bwd,
argmax backward, scale rows, permute, device CSR build / transpose / source
blocks, the CSR1 / FMAT1 device loaders.  Results are checked against the
oracle so the run is also a parity run under the sanitizer."""
import os
import sys
import tempfile

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2007_06354_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

n, m = 600, 9000
src, dst = P.synth_rmat(n, m, 0.57, 0.19, 0.19, 0.05, 0)
loops = np.arange(n, dtype=np.uint32)
src, dst = np.concatenate([src, loops]), np.concatenate([dst, loops])
E = len(src)
og = O.Graph(n, src, dst)
dcsr = P.build_csr(n, src, dst, P.DST_MAJOR)
scsr = P.transpose(n, n, *dcsr)
ok = {}


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


for long_thr in (0, 64):  # automatic plan, then hub rows as long-row units
    gd = P.Graph(*dcsr, orientation=P.DST_MAJOR)
    gs = P.Graph(*scsr, orientation=P.SRC_MAJOR)
    if long_thr:
        gd.set_plan(long_threshold=long_thr)
        gs.set_plan(long_threshold=long_thr)
        assert gd.num_long_rows > 0
    tag = f"thr{long_thr}"
    for F in (100, 256, 602):
        ld = (F + 3) // 4 * 4
        x = P.synth_normal(n, F, 1)
        gy = P.synth_normal(n, F, 3)
        w = P.synth_gcn_weights(n, src, dst)
        xb = torch.zeros((n, ld), device="cuda")
        xb[:, :F] = dev(x)
        xd = xb[:, :F]
        gb = torch.zeros((n, ld), device="cuda")
        gb[:, :F] = dev(gy)
        gyd = gb[:, :F]
        wd = dev(w)
        out = P.binary_reduce(gd, "u_mul_e_add_v", u=xd, e=wd)
        ok[f"{tag} F{F} u_mul_e"] = O.bit_equal(out.cpu().numpy(), O.binary_reduce(
            og, O.named_config("u_mul_e_add_v"), u=x, e=w))
        wp = gd.permute_edges(wd)
        out = P.binary_reduce(gd, "u_mul_e_add_v", u=xd, e=wp, e_order=P.EDGE_BY_POS)
        ok[f"{tag} F{F} u_mul_e by pos"] = O.bit_equal(out.cpu().numpy(), O.binary_reduce(
            og, O.named_config("u_mul_e_add_v"), u=x, e=w))
        gx = P.binary_reduce(gs, "v_mul_e_add_u", v=gyd, e=wd)
        ok[f"{tag} F{F} grad_x"] = O.bit_equal(gx.cpu().numpy(), O.sum_backward(og, gy, w))
        mean = torch.empty((n, F), device="cuda")
        mx, au, ae = P.binary_reduce(gd, "u_copy_max_v", u=xd, want_arg_other=True,
                                     want_arg_edge=True, out2=mean, reduce2=P.MEAN)
        v2, au2, ae2 = O.copy_max_argmax(og, x)
        ok[f"{tag} F{F} max+argmax+mean"] = (
            O.bit_equal(mx.cpu().numpy(), v2) and np.array_equal(au.cpu().numpy(), au2) and
            np.array_equal(ae.cpu().numpy(), ae2) and O.bit_equal(mean.cpu().numpy(), O.mean(og, x)))
        gmax = P.argmax_backward(au, gyd, n)
        ok[f"{tag} F{F} max bwd"] = O.max_rel_error(
            gmax.cpu().numpy(), O.argmax_backward(au2, gy, n)) <= 1e-6
        deg = np.diff(dcsr[0].astype(np.int64))
        inv = np.zeros(n, np.float32)
        inv[deg > 0] = np.float32(1) / deg[deg > 0].astype(np.float32)
        gm = P.binary_reduce(gs, (P.V, P.NONE, P.COPY, P.SUM, P.U), v=gyd, other_scale=dev(inv))
        ok[f"{tag} F{F} mean bwd"] = O.bit_equal(gm.cpu().numpy(), O.mean_backward(og, gy))
        gd.set_source_blocks(3)
        s3 = P.binary_reduce(gd, (P.U, P.NONE, P.COPY, P.MEAN, P.V), u=xd)
        gd.set_source_blocks(0)
        ok[f"{tag} F{F} mean, 3 source blocks"] = O.bit_equal(s3.cpu().numpy(), O.mean(og, x))
        if F == 100:
            v = P.synth_uniform(n, F, 7)
            for name in ("u_add_v_add_v", "u_mul_v_add_v", "u_dot_v_copy_e", "u_add_v_copy_e",
                         "e_copy_max_v", "u_copy_min_v"):
                e_full = P.synth_uniform(E, F, 9)
                got = P.binary_reduce(gd, name, u=xd, v=dev(v), e=dev(e_full))
                want = O.binary_reduce(og, O.named_config(name), u=x, v=v, e=e_full)
                ok[f"{tag} {name}"] = O.bit_equal(got.cpu().numpy(), want)
    # multi-head (cfg4 shape) fwd, grad_a, edge softmax
    H, D = 8, 16
    x = P.synth_normal(n, H * D, 1)
    gy = P.synth_normal(n, H * D, 3)
    logits = P.synth_normal(E, H, 2)
    a = P.edge_softmax(gd, dev(logits))
    ga = P.edge_softmax_backward(gd, a, dev(P.synth_normal(E, H, 4)))
    ok[f"{tag} softmax finite"] = bool(torch.isfinite(a).all() and torch.isfinite(ga).all())
    out = P.binary_reduce(gd, "u_mul_e_add_v", u=dev(x), e=a, heads=H)
    grad_a = P.binary_reduce(gd, (P.U, P.V, P.DOT, P.COPY_LAST, P.E), u=dev(x), v=dev(gy), heads=H)
    ok[f"{tag} multi-head finite"] = bool(torch.isfinite(out).all() and torch.isfinite(grad_a).all())
    gd.close()
    gs.close()

# device CSR build / transpose, the container loaders
sd, dd = dev(src.view(np.int32)), dev(dst.view(np.int32))
ip, ix, ei = P.build_csr_device(n, sd, dd, P.DST_MAJOR)
ok["build_csr_device"] = all(np.array_equal(a.cpu().numpy().view(np.uint32), b)
                             for a, b in zip((ip, ix, ei), dcsr))
tp = P.transpose_device(n, n, ip, ix, ei)
ok["transpose_device"] = all(np.array_equal(a.cpu().numpy().view(np.uint32), b)
                             for a, b in zip(tp, scsr))
P.validate_csr_device(n, n, ip, ix, ei)
d = tempfile.mkdtemp()
P.save_csr(d + "/g.csr", P.DST_MAJOR, n, n, *dcsr)
gl = P.Graph.load(d + "/g.csr")
xs = P.synth_normal(n, 32, 5)
ok["load_csr1"] = O.bit_equal(P.binary_reduce(gl, "u_copy_add_v", u=dev(xs)).cpu().numpy(),
                              O.binary_reduce(og, O.named_config("u_copy_add_v"), u=xs))
P.save_feature_matrix(d + "/x.fmat", xs)
ok["load_fmat1"] = np.array_equal(P.load_feature_matrix(d + "/x.fmat", device=0, ld=36).cpu().numpy(), xs)
torch.cuda.synchronize()
bad = [k for k, v in ok.items() if not v]
print(f"sanitize_case: {len(ok)} checks, {len(bad)} failed {bad}")
sys.exit(1 if bad else 0)
