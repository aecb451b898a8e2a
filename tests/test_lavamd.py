"""LavaMD (C4; not in the reference: the framework's restatement of Rodinia
lavaMD, SURVEY.md Appendix C — parity pinned only against our own oracle and
an independent numpy model)."""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_2308_16877_b200 import engine as E

STAT_FIELDS = ["total_invocations", "approx_invocations", "divergent_warp_steps", "total_warp_steps",
               "resident_warps"]


def numpy_lavamd(rv, qv, b1, P, alpha=0.5):
    """Independent model: all 27-neighbourhood box pairs, np.exp."""
    a2 = 2 * alpha * alpha
    nb = b1 ** 3
    fv = np.zeros((nb * P, 4))
    R = rv.reshape(nb, P, 4)
    Q = qv.reshape(nb, P)
    for b in range(nb):
        bx, by, bz = b % b1, (b // b1) % b1, b // (b1 * b1)
        for dz in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    x, y, z = bx + dx, by + dy, bz + dz
                    if not (0 <= x < b1 and 0 <= y < b1 and 0 <= z < b1):
                        continue
                    o = (z * b1 + y) * b1 + x
                    A, B, q = R[b], R[o], Q[o]
                    r2 = A[:, None, 0] + B[None, :, 0] - (A[:, None, 1:] * B[None, :, 1:]).sum(-1)
                    vij = np.exp(-a2 * r2)
                    fs = 2 * vij
                    d = A[:, None, 1:] - B[None, :, 1:]
                    fv[b * P:(b + 1) * P, 0] += (q[None, :] * vij).sum(1)
                    fv[b * P:(b + 1) * P, 1:] += (q[None, :, None] * fs[..., None] * d).sum(1)
    return fv


def test_lava_exp_accuracy():
    L = oracle.oracle()
    L.oracle_lava_exp.restype = C.c_double
    L.oracle_lava_exp.argtypes = [C.c_double]
    xs = np.linspace(-30, 30, 20001)
    got = np.array([L.oracle_lava_exp(x) for x in xs])
    rel = np.abs(got - np.exp(xs)) / np.exp(xs)
    assert rel.max() < 2e-15  # one-FMA reduction with rounded ln2 (|k| <= 44 here), degree-11 fit


def test_oracle_lavamd_matches_numpy_model():
    b1, P = 3, 32
    rv, qv = E.make_lavamd(b1, P, 7)
    fv = np.zeros((b1 ** 3 * P, 4))
    grid = E.GridConfig(b1 ** 3, P, 32, 1)
    reg = E.lavamd_region(rv, qv, fv, b1, P)
    rc, st, msg = oracle.oracle_run(grid, b1 ** 3, 1, reg, None)
    assert rc == 0, msg
    want = numpy_lavamd(rv, qv, b1, P)
    assert np.allclose(fv, want, rtol=1e-12, atol=1e-12)
    # 27 box-box rounds for the centre box, fewer at faces/edges/corners
    assert st.total_invocations == P * sum(
        sum(1 for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)
            if 0 <= b % b1 + dx < b1 and 0 <= (b // b1) % b1 + dy < b1 and 0 <= b // (b1 * b1) + dz < b1)
        for b in range(b1 ** 3))


def test_lavamd_rejects_ini_and_wrong_team_shape():
    b1, P = 2, 32
    rv, qv = E.make_lavamd(b1, P, 1)
    fv = np.zeros((b1 ** 3 * P, 4))
    reg = E.lavamd_region(rv, qv, fv, b1, P)
    with pytest.raises(E.ConfigError, match="trip count"):
        E.run_region(E.GridConfig(8, P, 32, 1), 8, 1, reg, E.perfo("ini", 20))
    with pytest.raises(E.ConfigError, match="particles"):
        E.run_region(E.GridConfig(8, 64, 32, 1), 8, 1, reg, None)


@pytest.mark.gpu
@pytest.mark.parametrize("spec_fn", [lambda: None, lambda: E.taf(2, 4, 0.05, "thread"),
                                     lambda: E.taf(2, 4, 0.05, "warp"), lambda: E.taf(3, 8, 0.1, "team"),
                                     lambda: E.taf(1, 2, 0.5, "warp"), lambda: E.perfo("small", 3),
                                     lambda: E.perfo("herded_large", 4, "warp")])
def test_cuda_lavamd_bit_exact_vs_oracle(spec_fn):
    import torch
    b1, P, ipt = 4, 64, 2
    nb = b1 ** 3
    rv, qv = E.make_lavamd(b1, P, 3)
    grid = E.GridConfig(nb // ipt, P, 32, ipt)
    fv = torch.zeros((nb * P, 4), dtype=torch.float64, device="cuda")
    paths = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    lr = E.run_region(grid, nb, 1, E.lavamd_region(torch.from_numpy(rv).cuda(), torch.from_numpy(qv).cuda(), fv, b1, P),
                      spec_fn(), paths=paths)
    ofv = np.zeros((nb * P, 4))
    op = np.zeros(nb, np.uint8)
    rc, st, msg = oracle.oracle_run(grid, nb, 1, E.lavamd_region(rv, qv, ofv, b1, P), spec_fn(), op)
    assert rc == 0, msg
    for f in STAT_FIELDS:
        assert lr.stats[f] == getattr(st, f), f
    assert np.array_equal(fv.cpu().numpy(), ofv)
    assert np.array_equal(paths.cpu().numpy(), op)


@pytest.mark.gpu
@pytest.mark.parametrize("b1", [16, 32])
def test_cuda_lavamd_tiled_box_order_equals_natural(b1, monkeypatch):
    """Whole-grid launches process boxes in 16/32-wide tile columns (L2 reuse
    of the neighbourhoods, csrc/engine_thread.cu lava_tile_order); teams are
    independent, so forces, stats and paths equal the natural order's."""
    import torch
    P = 128
    nb = b1 ** 3
    rv, qv = E.make_lavamd(b1, P, 11)
    d_rv, d_qv = torch.from_numpy(rv).cuda(), torch.from_numpy(qv).cuda()
    grid = E.GridConfig(nb, P, 32, 1)
    res = []
    for tile in ["1", "0"]:
        monkeypatch.setenv("HPAC_LAVA_TILE", tile)
        fv = torch.zeros((nb * P, 4), dtype=torch.float64, device="cuda")
        paths = torch.zeros(nb, dtype=torch.uint8, device="cuda")
        lr = E.run_region(grid, nb, 1, E.lavamd_region(d_rv, d_qv, fv, b1, P),
                          E.taf(3, 8, 0.1, "warp"), paths=paths)
        res.append((lr.stats, fv.cpu().numpy(), paths.cpu().numpy()))
    for f in STAT_FIELDS:
        assert res[0][0][f] == res[1][0][f], f
    assert np.array_equal(res[0][1], res[1][1])
    assert np.array_equal(res[0][2], res[1][2])
