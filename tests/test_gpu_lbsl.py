"""NEXT-3 LBSL on the GPU: one LBSL step applied to a device-resident jagged batch through
the C-ABI (uh_lbsl_select / uh_lbsl_rows on the host, uh_gather_rows on the device),
compared element by element (bit-exact: it is a copy) with the kept rows the ORACLE
(oracle/lbsl.py, Alg. 1) selects on the same seeded batch."""
import numpy as np
import pytest
import torch

import lbsl as OL
from paper_2602_16986_b200 import lbsl as NL
from paper_2602_16986_b200 import uhstu as U

pytestmark = pytest.mark.gpu


def _oracle_rows(B, dec, new, seed, rank, t):
    off = np.concatenate([[0], np.cumsum(B)]).astype(np.int64)
    rows = []
    for u in range(len(B)):
        pos = OL.sl_subset(B[u], new[u], seed, rank, t, u) if dec[u] == OL.TRUNCATED else range(B[u])
        rows += [off[u] + j for j in pos]
    return np.asarray(rows, np.int64)


@pytest.mark.parametrize("dtype,d", [(torch.bfloat16, 512), (torch.float32, 64), (torch.bfloat16, 8)])
def test_lbsl_apply_matches_oracle_rows(dtype, d):
    rng = np.random.default_rng(7)
    cfg = NL.LbslConfig(T_warm=2, T_recal=2, gamma=1.7, ell_sl=512, seed=31)
    rt = NL.LBSL(cfg, rank=3)
    st = OL.LbslState(OL.LbslParams(R=1, T_warm=2, T_recal=2, gamma=1.7, ell_sl=512, b=32))
    for t in range(1, 6):
        B = [int(min(16384, 256 * (1 + rng.pareto(1.5)))) for _ in range(32)]
        B[5] = 0
        jag = U.JaggedBatch.from_lengths(B)
        x = torch.randn(jag.T, d, device="cuda").to(dtype)
        # the oracle's step runs with rank 0 of an R = 1 world; the runtime's rank id only
        # selects the random stream, so compare against the oracle's rank_select at rank 3
        od, on = OL.rank_select(B, st.params, st.ell_bar, t > 2, 31, 3, t)
        OL.lbsl_step(st, [B], 31)
        jag2, y, dec = rt.apply(jag, x)
        torch.cuda.synchronize()
        assert list(dec) == od and list(jag2.lengths) == on
        want = x.cpu()[torch.from_numpy(_oracle_rows(B, od, on, 31, 3, t))]
        assert torch.equal(y.cpu(), want)


def test_gather_rows_edge_cases():
    x = torch.randn(100, 64, device="cuda", dtype=torch.bfloat16)
    empty = torch.zeros(0, dtype=torch.int32, device="cuda")
    assert U.gather_rows(empty, x).shape == (0, 64)
    rows = torch.tensor([99, 0, 0, 57], dtype=torch.int32, device="cuda")
    assert torch.equal(U.gather_rows(rows, x).cpu(), x.cpu()[[99, 0, 0, 57]])
    with pytest.raises(U.UhError):                         # 7 bf16 = 14 bytes per row
        U.gather_rows(rows, torch.zeros(100, 7, device="cuda", dtype=torch.bfloat16))
