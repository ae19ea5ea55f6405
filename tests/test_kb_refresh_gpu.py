"""Template refresh on the GPU: after profiling trials are recorded, the
refreshed engine's Monte Carlo samples equal the reference's
monte_carlo_remaining_demand on the updated reference graph (bit-exact)."""

import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def test_refresh_matches_reference_after_trials():
    import torch
    from tests.dispatch_hook import import_pdgsim
    try:
        import_pdgsim()
    except ImportError:
        pytest.skip("pdgsim not installed in baseline/_ref")
    from pdgsim.estimator import monte_carlo_remaining_demand as ref_mc
    from pdgsim.pdgraph import RateProfile
    from pdgsim.pdgraph import record_trial as ref_record
    from paper_2506_14851_b200.estimator import DemandEngine
    from paper_2506_14851_b200.graphs import record_trial
    from tests.kb_trials import setup
    base, kb, ref_trials, kb_trials = setup()
    eng = DemandEngine({"vc": kb})
    env = RateProfile()
    dev = eng.device

    def check(seed0):
        order = eng.bank.unit_order["vc"]
        gi, ui, sd = [], [], []
        for k, uid in enumerate(order):
            gi.append(0)
            ui.append(k)
            sd.append(seed0 + k)
        t = lambda a, dt: torch.tensor(a, dtype=dt, device=dev)  # noqa: E731
        res = eng.run(t(gi, torch.int32), t(ui, torch.int32), t(sd, torch.int64), n=512,
                      bucket_count=64, samples=True)
        S = res["samples"].cpu().numpy()
        for k, uid in enumerate(order):
            want = ref_mc(base, uid, [], env, 512, seed0 + k)
            assert _sha(S[k]) == _sha(want.samples), uid

    check(100)
    for i, (rt, kt) in enumerate(zip(ref_trials, kb_trials)):
        ref_record(base, rt)
        record_trial(kb, kt)
        if i % 20 == 19:
            eng.refresh("vc")
            check(200 + i)
