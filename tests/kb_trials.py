"""Shared setup for the template-refresh tests: a reference archetype graph,
its knowledge-base copy, and new profiling trials taken from a second
instance of the same archetype."""

from tests.dispatch_hook import import_pdgsim


def setup(kind="verify-chain", n_trials=60, trials=200, capacity=220):
    import_pdgsim()
    from pdgsim.pdgraph import graph_to_dict
    from pdgsim.workload import archetype
    from paper_2506_14851_b200.graphs import KBRecord, graph_from_kb
    base = archetype(kind, {"trials": trials, "bucket_count": 64, "app_id": kind,
                            "capacity": capacity}, seed=1)
    src = archetype(kind, {"trials": trials, "bucket_count": 64, "app_id": kind,
                           "capacity": capacity}, seed=9)
    kb = graph_from_kb(graph_to_dict(base))
    by_trial: dict = {}
    for uid, u in src.units.items():
        for r in u.records:
            by_trial.setdefault(r.trial_id, {})[uid] = r
    ref_trials = [by_trial[t] for t in sorted(by_trial)][:n_trials]
    kb_trials = [{uid: KBRecord(1000 + i, r.input_len, r.output_len, r.parallelism,
                                r.duration, r.next_unit) for uid, r in tr.items()}
                 for i, tr in enumerate(ref_trials)]
    from pdgsim.pdgraph import UnitRecord
    ref_trials = [{uid: UnitRecord(1000 + i, r.input_len, r.output_len, r.parallelism,
                                   r.duration, r.next_unit) for uid, r in tr.items()}
                  for i, tr in enumerate(ref_trials)]
    return base, kb, ref_trials, kb_trials
