"""Records, on every PriorityRefresh of a reference simulation, the task
table the preemption + dispatch decisions were made on and the actions the
reference took (simcore.py:636-687, 512-516), so a planner can be checked
against the reference on real simulator states."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def import_pdgsim():
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(path) and path not in sys.path:
            sys.path.insert(0, path)
    import pdgsim  # noqa: F401
    return pdgsim


class _RecList(list):
    def __init__(self, items, log):
        super().__init__(items)
        self.log = log

    def append(self, task):
        self.log.append((1, task.key_id))
        super().append(task)


def record_config1(max_refreshes=None):
    """Run BASELINE config 1 under the reference; returns a list of
    (table, slots, hysteresis, actions) per PriorityRefresh that preempted
    or dispatched.  table = dict of task arrays; actions = [(kind, task)]."""
    import_pdgsim()
    from pdgsim import simcore
    from pdgsim.prewarm import CachePolicy
    from pdgsim.sched import Policy
    from pdgsim.workload import archetype, generate

    code_gen = archetype("code-check", {"trials": 200, "bucket_count": 64, "scale": 0.6,
                                        "app_id": "code-gen"}, seed=3)
    fact = archetype("verify-chain", {"trials": 200, "bucket_count": 64,
                                      "app_id": "fact-verify"}, seed=1)
    wl = generate({"small": 1.0}, 1000, 1000.0, seed=0,
                  class_apps={"small": ["code-gen", "fact-verify"]})
    cfg = simcore.SimConfig(bucket_count=64, mc_samples=512,
                            cache_policy=CachePolicy.HERMES_PLAN)
    out = []
    state = {}
    Sim = simcore.Simulator
    orig_preempt, orig_start, orig_refresh = Sim._preempt, Sim._start_task, Sim._on_PriorityRefresh

    def snap(self):
        tasks = []
        for b, be in enumerate(self.backends.values()):
            tasks += [(b, 0, t) for t in be.queue]
            tasks += [(b, 1, t) for t in be.active.values()]
        apps = sorted({(t.app.inst.arrival_time, t.app.inst.app_instance_id)
                       for _, _, t in tasks})
        rank = {a: i for i, a in enumerate(apps)}
        table = {"backend": [b for b, _, _ in tasks], "active": [a for _, a, _ in tasks],
                 "key": [self.prio[t.app.inst.app_instance_id].key for _, _, t in tasks],
                 "app_rank": [rank[(t.app.inst.arrival_time, t.app.inst.app_instance_id)]
                              for _, _, t in tasks],
                 "stage": [t.stage_index for _, _, t in tasks],
                 "request": [t.request_index for _, _, t in tasks]}
        ids = {t.key_id: i for i, (_, _, t) in enumerate(tasks)}
        log = []
        for be in self.backends.values():
            be.queue = _RecList(be.queue, log)
        state.update(table=table, ids=ids, log=log,
                     slots=[be.slots for be in self.backends.values()])

    def preempt(self):
        snap(self)
        return orig_preempt(self)

    def start(self, backend, task):
        if "log" in state:
            state["log"].append((2, task.key_id))
        return orig_start(self, backend, task)

    def refresh(self):
        state.clear()
        r = orig_refresh(self)
        if "log" in state:
            acts = [(k, state["ids"][kid]) for k, kid in state["log"]]
            if acts and (max_refreshes is None or len(out) < max_refreshes):
                out.append((state["table"], state["slots"],
                            self.cfg.preemption_hysteresis, acts))
            for be in self.backends.values():
                be.queue = list(be.queue)
        state.clear()
        return r

    Sim._preempt, Sim._start_task, Sim._on_PriorityRefresh = preempt, start, refresh
    try:
        simcore.run_simulation({"code-gen": code_gen, "fact-verify": fact}, wl,
                               Policy.GITTINS, cfg, seed=0)
    finally:
        Sim._preempt, Sim._start_task, Sim._on_PriorityRefresh = (orig_preempt, orig_start,
                                                                  orig_refresh)
    return out
