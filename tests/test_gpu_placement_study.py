"""The placement study (BASELINE.json configs[4]) at test scale: every mode's
final grid matches the oracle on the final simulation state, and the solver's
trajectory is bit-identical with the analysis lockstep, asynchronous (snapshot
or in place) or on another GPU -- the analysis never writes simulation data
(SPEC.md:464)."""
import pytest

pytestmark = pytest.mark.gpu


_LOCKSTEP = {}


def _run(mode):
    from tools import placement_study as ps
    return ps.run_fanin(1_000_003, 6) if mode == "fanin" else ps.run_mode(mode, 1_000_003, 6)


@pytest.mark.parametrize("mode", ["lockstep", "async_snapshot", "async_inplace", "peer", "fanin"])
def test_placement_mode_agrees_and_does_not_interfere(cuda_available, mode):
    """One placement mode vs the oracle and vs the lockstep trajectory.  The
    peer and fan-in modes need a second GPU: on a 1-GPU box they SKIP (visibly)."""
    if not cuda_available:
        pytest.fail("needs a CUDA device")
    import torch

    from tools import placement_study as ps
    if mode in ("peer", "fanin") and torch.cuda.device_count() < 2:
        pytest.skip(f"placement mode {mode!r} needs >= 2 GPUs (this box has {torch.cuda.device_count()})")
    if "lockstep" not in _LOCKSTEP:
        _LOCKSTEP["lockstep"] = _run("lockstep")
    results = [_LOCKSTEP["lockstep"]] if mode == "lockstep" else [_LOCKSTEP["lockstep"], _run(mode)]
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
