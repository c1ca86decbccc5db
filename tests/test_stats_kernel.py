"""The statistics pass through the C-ABI on synthetic response rows (GPU).

cs_rep_stats replaces responses.mean() per replication and the order
statistics np.quantile interpolates over each point's merged responses
(sim.py:406-438).  These rows stress the row pass's inside-bracket staging
and hand-over path (csrc/stats.cu row_stats_kernel): heavy ties that put a
large share of every row inside a bracket (staging rings fill every leaf
group, candidate lists overflow and the brackets widen), strongly
autocorrelated rows (inside values cluster in a lane's leaf), and row
lengths that leave remainder leaves.  Per-row means must be bit-exact with
numpy's pairwise sum, order statistics bit-exact with np.sort.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu


def _ranks(n: int) -> list[int]:
    out = set()
    for q in (0.5, 0.95, 0.99):
        x = q * (n - 1)
        out.update((int(np.floor(x)), int(np.ceil(x))))
    return sorted(out)


def _rows(kind: str, G: int, R: int, m: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    if kind == "ties":  # five values: every target sits inside a huge tie block
        vals = np.array([0.5, 1.0, 1.5, 2.0, 3.0])
        return vals[rng.choice(5, size=(G, R, m), p=[0.1, 0.3, 0.35, 0.2, 0.05])]
    if kind == "ar1":  # log-AR(1), phi = 0.999: long runs of near-equal responses
        z = rng.standard_normal((G, R, m))
        x = np.empty_like(z)
        x[..., 0] = z[..., 0]
        for i in range(1, m):
            x[..., i] = 0.999 * x[..., i - 1] + 0.0447 * z[..., i]
        return np.exp(x)
    return rng.exponential(1.0, size=(G, R, m)) + rng.random((G, R, 1))  # shifted per row


@pytest.mark.parametrize("kind,m", [("ties", 40_000), ("ar1", 40_000), ("exp", 33_333), ("exp", 7)])
def test_rep_stats_synthetic_rows(kind, m):
    import torch

    import paper_2604_14993_b200._native as N

    lib = N.load()
    G, R = 3, (48 if m > 100 else 200_000)
    host = _rows(kind, G, R, m, seed=11 + m)
    ldr = (m + 15) // 16 * 16
    buf = np.zeros((G * R, ldr), np.float64)
    buf[:, :m] = host.reshape(G * R, m)
    d_resp = torch.from_numpy(buf).cuda()
    d_summ = torch.zeros(G * R * C.sizeof(N.RepSummary), dtype=torch.uint8, device="cuda")
    n = R * m
    rk = _ranks(n)
    ranks = np.array(rk * G, np.int64)
    out = np.zeros(len(ranks), np.float64)
    st = torch.cuda.current_stream()
    rc = lib.cs_rep_stats(d_resp.data_ptr(), G, R, m, ldr, d_summ.data_ptr(), N.ptr(ranks, C.c_int64), len(rk),
                          N.ptr(out, C.c_double), None, st.cuda_stream)
    N.check(rc, "cs_rep_stats")
    summ = d_summ.cpu().numpy().view(N.SUMMARY_DTYPE).reshape(G, R)
    for g in range(G):
        means = np.array([row.mean() for row in host[g]])
        assert np.array_equal(bits(summ[g]["resp_mean"]), bits(means)), (kind, g)
        merged = np.sort(host[g].ravel())
        for i, r in enumerate(rk):
            assert bits(out[g * len(rk) + i]) == bits(merged[r]), (kind, g, r)
