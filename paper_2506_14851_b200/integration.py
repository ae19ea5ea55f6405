"""Drop the GPU hot path into the reference simulator (``pdgsim``).

The reference has no plugin registry: ``simcore.py`` imports the hot-path
functions by name (simcore.py:20-40) and ``sched.refresh_priorities`` calls
``gittins_rank_batch`` as a module global (sched.py:294).  ``patch_pdgsim``
rebinds exactly those names (the same seam SURVEY.md 8(b) lists):

    pdgsim.sched.gittins_rank_batch            -> K1a  (also used by gittins_rank_points)
    pdgsim.simcore.refresh_priorities          -> a2 batched refresh over K1a
    pdgsim.simcore.monte_carlo_remaining_demand -> K2/K3 engine
    pdgsim.simcore.plan_prewarm                -> K4a
    pdgsim.sched.ApplicationInstance.set_remaining -> a4 (GPU bucketing)

and makes the drop-in return ``pdgsim.estimator.RemainingDemand`` objects;
``restore`` undoes it.
"""

from __future__ import annotations

from . import estimator as _est
from . import prewarm as _pw
from . import sched as _sched

_SAVED: dict = {}


def patch_pdgsim(pdgsim) -> None:
    sched, simcore = pdgsim.sched, pdgsim.simcore
    if _SAVED:
        return
    _SAVED.update({
        (sched, "gittins_rank_batch"): sched.gittins_rank_batch,
        (simcore, "refresh_priorities"): simcore.refresh_priorities,
        (simcore, "monte_carlo_remaining_demand"): simcore.monte_carlo_remaining_demand,
        (simcore, "plan_prewarm"): simcore.plan_prewarm,
        (sched.ApplicationInstance, "set_remaining"): sched.ApplicationInstance.set_remaining,
    })
    _SAVED[(_est, "RESULT_TYPE")] = _est.RESULT_TYPE
    _est.RESULT_TYPE = pdgsim.estimator.RemainingDemand     # the reference's own result type
    sched.gittins_rank_batch = _sched.gittins_rank_batch
    simcore.refresh_priorities = _sched.refresh_priorities
    simcore.monte_carlo_remaining_demand = _est.monte_carlo_remaining_demand
    simcore.plan_prewarm = _pw.plan_prewarm

    def set_remaining(self, remaining, bucket_count):
        _sched.set_remaining(self, remaining, bucket_count)

    sched.ApplicationInstance.set_remaining = set_remaining


def restore() -> None:
    for (obj, name), fn in _SAVED.items():
        setattr(obj, name, fn)
    _SAVED.clear()
