"""The placement study (BASELINE.json configs[4]) at test scale: every mode's
final grid matches the oracle on the final simulation state, and the solver's
trajectory is bit-identical with the analysis lockstep, asynchronous (snapshot
or in place) or on another GPU -- the analysis never writes simulation data
(SPEC.md:464)."""
import pytest

pytestmark = pytest.mark.gpu


def test_placement_modes_agree_and_do_not_interfere(cuda_available):
    if not cuda_available:
        pytest.fail("needs a CUDA device")
    import torch

    from tools import placement_study as ps
    modes = [m for m in ps.MODES if m not in ("peer", "fanin") or torch.cuda.device_count() > 1]
    results = [ps.run_fanin(1_000_003, 6) if m == "fanin" else ps.run_mode(m, 1_000_003, 6) for m in modes]
    assert ps.check(results)
    for m, _, _ in results:
        assert m["solver_ms_per_step"] > 0 and m["actual_insitu_ms_per_step"] > 0


def test_direct_sum_study_modes_agree(cuda_available):
    """Compute-bound producer (O(N^2) direct sum) + the fused paper step, lockstep
    and asynchronous: identical trajectories, grids equal to the oracle."""
    if not cuda_available:
        pytest.fail("needs a CUDA device")
    from tools import insitu_direct_study as ds
    results = [ds.run(m, 4099, 4) for m in ("lockstep", "async_snapshot", "async_inplace")]
    assert ds.check(results)
