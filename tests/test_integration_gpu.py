"""End-to-end drop-in: the reference simulator (pdgsim, pip-installed into
baseline/_ref) runs BASELINE config 1 with its hot path (Gittins batch,
refresh, Monte Carlo engine, set_remaining bucketing, prewarm planner)
replaced by the GPU path; the event log must be byte-identical to the one
the unmodified reference produced (sha256 recorded in tests/golden)."""

import hashlib
import os
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _pdgsim():
    if os.path.isdir(REF) and REF not in sys.path:
        sys.path.insert(0, REF)
    try:
        import pdgsim
    except ImportError:
        pytest.skip("pdgsim not installed in baseline/_ref")
    return pdgsim


def test_config1_simulation_byte_identical(config1_golden):
    pdgsim = _pdgsim()
    from pdgsim import simcore
    from pdgsim.prewarm import CachePolicy
    from pdgsim.sched import Policy
    from pdgsim.workload import archetype, generate

    from paper_2506_14851_b200 import integration
    code_gen = archetype("code-check", {"trials": 200, "bucket_count": 64, "scale": 0.6,
                                        "app_id": "code-gen"}, seed=3)
    fact = archetype("verify-chain", {"trials": 200, "bucket_count": 64,
                                      "app_id": "fact-verify"}, seed=1)
    wl = generate({"small": 1.0}, 1000, 1000.0, seed=0,
                  class_apps={"small": ["code-gen", "fact-verify"]})
    cfg = simcore.SimConfig(bucket_count=64, mc_samples=512,
                            cache_policy=CachePolicy.HERMES_PLAN)
    integration.patch_pdgsim(pdgsim)
    try:
        assert pdgsim.simcore.monte_carlo_remaining_demand.__module__.startswith(
            "paper_2506_14851_b200")
        res = simcore.run_simulation({"code-gen": code_gen, "fact-verify": fact}, wl,
                                     Policy.GITTINS, cfg, seed=0)
    finally:
        integration.restore()
    sha = hashlib.sha256("\n".join(res.event_log).encode()).hexdigest()
    assert len(res.event_log) == config1_golden["event_log_lines"]
    assert sha == config1_golden["event_log_sha256"]
