"""GEMM engines on the B200: TMA-fed tcgen05 bf16x3 (default), the gather
tcgen05 engine and exact fp32 SIMT,
against a float64 numpy product, over the operand orientations and ragged
shapes the training step uses (tolerances stated per engine)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2307_07649_b200 as T

pytestmark = pytest.mark.gpu

SHAPES = [(300, 200, 472), (128, 100, 64), (1, 100, 1200), (1800, 300, 100), (77, 472, 333),
          (2845, 572, 200), (13, 16, 8)]


@pytest.mark.parametrize("impl,tol", [(T.GEMM_TMA, 3e-5), (T.GEMM_SIMT, 2e-6), (T.GEMM_GATHER, 3e-5)])
@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("at,bt", [(False, True), (True, False), (False, False), (True, True)])
def test_gemm_engine(impl, tol, M, N, K, at, bt):
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.normal(size=(M, K))
    B = rng.normal(size=(K, N))
    ref = A @ B
    Ain = A.T.copy() if at else A
    Bin = B.T.copy() if bt else B
    for splits in (1, 3):
        C = T.debug_gemm(Ain, Bin, impl=impl, a_trans=at, b_trans=bt, splits=splits)
        err = np.abs(C - ref).max() / np.abs(ref).max()
        assert err < tol, (impl, M, N, K, at, bt, splits, err)
