"""K6: online-refinement event stream over a device-resident queue
(BASELINE config 4).

The reference re-estimates an application when one of its units completes:
``_complete_unit`` (simcore.py:562-587) records the observation, runs
``_estimate`` for the next unit (monte_carlo_remaining_demand with the
observations, estimator.py:305-362) and immediately refreshes that app's
priority (``_refresh([app], force=True)``).  Here completions arrive as
micro-batches of events; each batch is one engine launch (K3 conditioning +
K2 walk + bucketing, one warp per event) writing the apps' histogram rows in
place, one K1 launch over exactly those rows, and optionally a re-sort of the
whole queue's keys (K5) so the new ranks are visible in the global order.
"""

from __future__ import annotations

from typing import Optional

import torch

from . import _lib
from .estimator import DemandEngine
from .queue import HistQueue


class RefinementStream:
    def __init__(self, engine: DemandEngine, queue: HistQueue, graph_idx: torch.Tensor,
                 unit_idx: torch.Tensor, *, n_samples: int = 512, bucket_count: int = 256,
                 visit_cap: int = 64, penalty: float = 2.0):
        self.eng = engine
        self.q = queue
        self.graph_idx = graph_idx
        self.unit_idx = unit_idx
        self.n = int(graph_idx.numel())
        self.n_samples = n_samples
        self.bucket_count = bucket_count
        self.visit_cap = visit_cap
        self.penalty = penalty
        dev = queue.lo.device
        L = _lib.lib()
        tb = int(L.pdg_order_temp_bytes(self.n))
        self._temp = torch.empty(max(tb, 16), dtype=torch.uint8, device=dev)
        self.order_keys = torch.empty(self.n, dtype=torch.int64, device=dev)
        self.order_slots = torch.empty(self.n, dtype=torch.int32, device=dev)
        self._keys2 = torch.empty_like(self.order_keys)
        self._slots2 = torch.empty_like(self.order_slots)
        self._mark = torch.zeros(self.n, dtype=torch.uint8, device=dev)
        self._slots = torch.arange(self.n, dtype=torch.int32, device=dev)
        self._utemp = None
        self._ordered = False          # order_* hold the order of the current keys

    def process(self, app: torch.Tensor, next_unit: torch.Tensor, seed: torch.Tensor,
                obs_unit: Optional[torch.Tensor] = None, obs_val: Optional[torch.Tensor] = None,
                attained: Optional[torch.Tensor] = None, resort: bool = True, stream=None):
        """Apply one micro-batch of unit-completion events (device tensors):
        app int32[m] queue rows, next_unit int32[m] (local unit index), seed
        int64[m], obs_unit int32[m] (observed upstream local index or -1),
        obs_val f64[m,3], attained f64[m] (attained service at the event; it
        becomes the estimate age, sched.py:172).  Apps must be distinct
        within a batch."""
        m = int(app.numel())
        if m == 0:
            return
        self.unit_idx.index_copy_(0, app.long(), next_unit)
        g = self.graph_idx.index_select(0, app.long())
        self.eng.run(g, next_unit, seed, obs_unit, obs_val, n=self.n_samples,
                     bucket_count=self.bucket_count, visit_cap=self.visit_cap, queue=self.q,
                     slots=app, stream=stream)
        if attained is not None:
            self.q.est_age.index_copy_(0, app.long(), attained)
            self.q.age.index_copy_(0, app.long(), attained)
        self.q.score(self.penalty, rows=app, stream=stream)
        if resort and self._ordered:
            self._update_order(app, stream)     # K5b: merge the batch into the order
        elif resort:
            self.order(stream)
        else:
            self._ordered = False

    def order(self, stream=None) -> torch.Tensor:
        """Global order of the whole queue: full sort of the packed
        (key, arrival position) words."""
        L = _lib.lib()
        _lib.check(L.pdg_order(_lib.ptr(self.q.keys), _lib.ptr(self.order_keys),
                               _lib.ptr(self._slots), _lib.ptr(self.order_slots), self.n, 0,
                               _lib.ptr(self._temp), self._temp.numel(),
                               _lib.stream_ptr(stream)), "pdg_order")
        self._ordered = True
        return self.order_slots

    def _update_order(self, rows: torch.Tensor, stream=None) -> None:
        L = _lib.lib()
        m = int(rows.numel())
        need = int(L.pdg_order_update_temp_bytes(self.n, m))
        if self._utemp is None or self._utemp.numel() < need:
            self._utemp = torch.empty(need, dtype=torch.uint8, device=self.order_keys.device)
        _lib.check(L.pdg_order_update(
            _lib.ptr(self.q.keys), _lib.ptr(self.order_keys), _lib.ptr(self.order_slots), self.n,
            _lib.ptr(rows), m, _lib.ptr(self._mark), _lib.ptr(self._keys2),
            _lib.ptr(self._slots2), _lib.ptr(self._utemp), self._utemp.numel(),
            _lib.stream_ptr(stream)), "pdg_order_update")
        self.order_keys, self._keys2 = self._keys2, self.order_keys
        self.order_slots, self._slots2 = self._slots2, self.order_slots
