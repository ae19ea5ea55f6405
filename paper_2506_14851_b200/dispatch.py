"""K6 host side: the dispatch / preemption plan of one PriorityRefresh
(simcore.py:636-644 -> _preempt 652-687, _dispatch 512-516) computed on the
device from the task table; the caller applies the events in order.

Task order is the reference's _task_sort_key (simcore.py:339-344):
(Priority.key, arrival_time, app_instance_id, stage_index, request_index),
with (arrival_time, app_instance_id) passed as the app's arrival rank.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib

PREEMPT, START = 1, 2


class DispatchPlanner:
    def __init__(self, device: str = "cuda"):
        _lib.lib()
        self.device = torch.device(device)
        self._temp = None

    def plan(self, backend, active, key, app_rank, stage, request, slots,
             hysteresis: float = 1.5, preempt: bool = True, stream=None):
        """All task arrays are device tensors of one length (int32 / uint8 /
        float64 / int32(app_rank as uint32) / int32 / int32); slots is a list
        of per-backend slot counts.  Returns [(kind, task)] in apply order."""
        n = int(backend.numel())
        nb = len(slots)
        if nb < 1 or max(slots) > 1024 or min(slots) < 0:
            raise ValueError("1 <= backends, 0 <= slots <= 1024")
        L = _lib.lib()
        need = int(L.pdg_dispatch_temp_bytes(n, nb))
        if self._temp is None or self._temp.numel() < need:
            self._temp = torch.empty(need, dtype=torch.uint8, device=self.device)
        cap = 3 * max(max(slots), 1)
        ev_task = torch.empty(nb * cap, dtype=torch.int32, device=self.device)
        ev_kind = torch.empty(nb * cap, dtype=torch.uint8, device=self.device)
        ev_count = torch.zeros(2 * nb, dtype=torch.int32, device=self.device)
        sl = torch.tensor(list(slots), dtype=torch.int32, device=self.device)
        _lib.check(L.pdg_dispatch_plan(
            _lib.ptr(backend), _lib.ptr(active), _lib.ptr(key), _lib.ptr(app_rank),
            _lib.ptr(stage), _lib.ptr(request), n, _lib.ptr(sl), nb, float(hysteresis),
            1 if preempt else 0, cap, _lib.ptr(ev_task), _lib.ptr(ev_kind), _lib.ptr(ev_count),
            _lib.ptr(self._temp), self._temp.numel(), _lib.stream_ptr(stream)),
            "pdg_dispatch_plan")
        st = np.zeros(1, dtype=np.int32)
        _lib.check(L.pdg_dispatch_status(_lib.ptr(self._temp), n, nb,
                                         st.ctypes.data_as(C.c_void_p), _lib.stream_ptr(stream)),
                   "pdg_dispatch_status")
        torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
        if st[0] == 1:
            raise ValueError("a backend has more running tasks than slots")
        if st[0] == 2:
            raise RuntimeError("dispatch plan needed more than 2 * slots waiting candidates")
        cnt = ev_count.cpu().numpy()
        # read back only the events each backend wrote (the rest of its
        # cap-sized region is never initialised)
        tk, kd = [], []
        for b in range(nb):
            used = int(cnt[b] + cnt[nb + b])
            tk.append(ev_task[b * cap:b * cap + used].cpu().numpy())
            kd.append(ev_kind[b * cap:b * cap + used].cpu().numpy())
        ev = []
        for b in range(nb):
            ev += [(int(kd[b][i]), int(tk[b][i])) for i in range(cnt[b])]
        for b in range(nb):
            ev += [(int(kd[b][cnt[b] + i]), int(tk[b][cnt[b] + i])) for i in range(cnt[nb + b])]
        return ev
