"""nmg_solve's active-set compaction: RHS that reached the stop rule leave the cycling
batch, the rest are gathered into a smaller batch (the RHS are independent).  The
per-RHS stopping cycles, residual histories and iterates must match the whole-batch solve (the
arithmetic of one RHS does not depend on the batch it runs in; the 1D fp64 residual switches from
the Ozaki to the DMMA kernel below 64 RHS, hence 1e-12 rather than bitwise) and the oracle's
stopping cycles."""
import numpy as np
import pytest

import nmg_inputs as ni
from tests._setup import gpu_hierarchy, oracle_hierarchy, weights_for

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import nmg_oracle as O  # noqa: E402

DEV = torch.device("cuda:0")


def _solve(cfg, f, W, y, tol, max_cycles, mode):
    h = gpu_hierarchy(cfg, f, W, max_rhs=y.shape[0], tuning={"no_compaction": mode})
    yd = torch.tensor(y, dtype=torch.float64, device=DEV)
    xd = torch.zeros_like(yd)
    rep = h.solve(yd, xd, tol=tol, max_cycles=max_cycles)
    torch.cuda.synchronize()
    return rep, xd.cpu().numpy()


@pytest.mark.parametrize("dim", [1, 2])
def test_compaction_matches_whole_batch(dim):
    if dim == 1:
        cfg = ni.CONFIGS[1].replace(n=512, levels=3, nrhs=40, alpha=1e-2)
        W = weights_for(cfg, "lin")
    else:
        cfg = ni.CONFIGS[2].replace(n=64, levels=3, nrhs=10)
        W = weights_for(cfg, "seed")
    f = ni.operator_factors(cfg)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha)
    cyc = 6
    # a stop tolerance inside the spread of the residuals after three cycles, so the RHS stop at
    # different cycles and the batch is compacted several times
    rep0, _ = _solve(cfg, f, W, y, 1e-300, cyc, 1)
    tol = float(np.median(rep0["history"][:, 3]))
    full, x_full = _solve(cfg, f, W, y, tol, cyc, 1)
    comp, x_comp = _solve(cfg, f, W, y, tol, cyc, 2)
    assert len(set(full["cycles"].tolist())) >= 2, full["cycles"]
    assert np.array_equal(full["cycles"], comp["cycles"])
    assert np.array_equal(full["converged"], comp["converged"])
    hf, hc = full["history"], comp["history"]
    assert np.array_equal(np.isnan(hf), np.isnan(hc))
    m = ~np.isnan(hf)
    assert np.max(np.abs(hf[m] - hc[m]) / hf[m]) < 1e-12
    for b in range(cfg.nrhs):
        nb = np.linalg.norm(x_full[b])
        assert np.linalg.norm(x_comp[b] - x_full[b]) <= 1e-12 * nb, b
    # the oracle stops every RHS at the same cycle (reading R13: +-1 only at the tolerance edge)
    H = oracle_hierarchy(cfg, f, W)
    orc = O.solve(H, y, tol=tol, max_cycles=cyc)
    assert np.max(np.abs(np.asarray(orc.cycles) - comp["cycles"])) <= 1
