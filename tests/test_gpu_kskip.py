"""Zero-block K skipping in the operator contractions is exact ("zero K blocks").

The Gaussian operators (BASELINE: sigma = 0.02, A = K^T K + alpha I) decay
below 2^-49 of their row maximum a few hundred grid points off the diagonal.  There every int8
truncation digit of the fp64 Ozaki residual's operator (ozaki.cu) and every f16 hi/lo value of
the FP16x3 apply's operator (gemm_tc.cu) is zero, and the kernels skip those K blocks.  The
skipped products are exact zeros, so the default path must be BITWISE the dense-K path
(nmg_tuning.dense_k = 1): same iterates, same fp64 residual histories, at the bench shapes
(config 1: Ozaki with > 64 RHS, 256- and 64-wide FP16x3 tiles; configs 2-4: both Ozaki passes).
"""
import numpy as np
import pytest

import nmg_inputs as ni
from tests._setup import gpu_hierarchy, weights_for

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _run(cfg, dense, cycles):
    f = ni.operator_factors(cfg)
    W = weights_for(cfg, "seed")
    h = gpu_hierarchy(cfg, f, W, max_rhs=cfg.nrhs, tuning={"dense_k": 1} if dense else None)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha)
    yd = torch.tensor(y, dtype=torch.float64, device="cuda")
    xd = torch.zeros_like(yd)
    rep = h.solve(yd, xd, tol=1e-300, max_cycles=cycles)
    return xd.cpu().numpy(), np.asarray(rep["history"])


@pytest.mark.parametrize("cid,over", [
    (1, dict(nrhs=1024)),                      # the bench batch: 4 lanes, tc_gemm<256, MC>, Ozaki
    (1, dict(nrhs=96)),                        # 64-wide FP16x3 tiles, Ozaki (> 64 RHS)
    (2, dict(nrhs=4)),
    (3, dict(nrhs=2)),
    (4, dict(nrhs=1)),
])
def test_kskip_bitwise_equal_dense(cid, over):
    cfg = ni.CONFIGS[cid].replace(**over)
    cycles = 2 if cfg.dim == 1 else 1
    x0, h0 = _run(cfg, False, cycles)
    x1, h1 = _run(cfg, True, cycles)
    assert np.array_equal(h0, h1, equal_nan=True), np.nanmax(np.abs(h0 - h1))
    assert np.array_equal(x0, x1), np.abs(x0 - x1).max()
