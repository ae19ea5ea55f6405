"""a11b on the GPU: HistQueue.update_attained (pdg_attained_service) equals the
oracle's restatement of Simulator._update_attained (simcore.py:306-313) bit
for bit (the oracle is pinned to the reference in tests/test_attained_cpu.py)."""

import numpy as np
import pytest

from tests.test_attained_cpu import oracle_of, random_tables

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed,n_apps,n_tasks", [(0, 50, 400), (1, 1, 0), (2, 3000, 20000)])
def test_update_attained_bit_exact(seed, n_apps, n_tasks):
    import torch
    from paper_2506_14851_b200.queue import HistQueue
    now, completed, progress, app, start, cold, service, active = random_tables(
        seed, n_apps, n_tasks)
    q = HistQueue(n_apps + 5, 16)
    q.n = n_apps
    d = lambda x, dt: torch.tensor(np.asarray(x), dtype=dt, device="cuda")  # noqa: E731
    q.update_attained(d(completed, torch.float64), d(progress, torch.float64),
                      d(app, torch.int32), d(active, torch.uint8), d(start, torch.float64),
                      d(cold, torch.float64), d(service, torch.float64), now)
    got = q.age[:n_apps].cpu().numpy()
    want = np.array(oracle_of(now, completed, progress, app, start, cold, service, active))
    assert np.array_equal(got, want)


def test_update_attained_rejects_bad_columns():
    import torch
    from paper_2506_14851_b200.queue import HistQueue
    q = HistQueue(8, 16)
    q.n = 4
    z = torch.zeros(4, dtype=torch.float64, device="cuda")
    t = torch.zeros(2, dtype=torch.float64, device="cuda")
    with pytest.raises(TypeError):
        q.update_attained(z, z, torch.zeros(2, dtype=torch.int64, device="cuda"),
                          torch.ones(2, dtype=torch.uint8, device="cuda"), t, t, t, 1.0)
