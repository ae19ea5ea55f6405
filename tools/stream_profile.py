"""Per-stage device timing of the config-4 refinement stream (development
tool): engine / K1 / re-sort per 1000-event batch over a 1M-app queue."""

import gzip
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import bench
    from paper_2506_14851_b200.estimator import DemandEngine
    from paper_2506_14851_b200.graphs import graph_from_kb
    from paper_2506_14851_b200.queue import HistQueue
    from paper_2506_14851_b200.stream import RefinementStream
    from tools import synth
    dev = torch.device("cuda", 0)
    n_apps, n_events, batch = 1_000_000, 20_000, 1000
    with gzip.open(os.path.join(ROOT, "tests", "golden", "graphs.json.gz"), "rt") as fh:
        docs = json.load(fh)
    graphs = {k: graph_from_kb(docs[k]) for k in bench.STREAM_TEMPLATES}
    q = synth.template_queue(graphs, n_apps, seed=41)
    ev = synth.events(graphs, q, n_events, seed=42)
    eng = DemandEngine(graphs, device=str(dev))
    hq = HistQueue(n_apps, 256)
    gi = torch.from_numpy(q["graph"]).to(dev)
    ui = torch.from_numpy(q["unit"].copy()).to(dev)
    seeds = torch.arange(n_apps, dtype=torch.int64, device=dev) * 1000003
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.run(gi, ui, seeds, n=512, bucket_count=256, queue=hq)
    e1.record()
    torch.cuda.synchronize()
    full = e0.elapsed_time(e1)
    hq.n = n_apps
    hq.score()
    st = RefinementStream(eng, hq, gi, ui, bucket_count=256)
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev)
         for k, v in (("app", ev["app"]), ("next", ev["next"]), ("comp", ev["completed"]),
                      ("obs", ev["obs"]), ("seed", ev["seed"]))}
    att = torch.full((n_events,), 5.0, dtype=torch.float64, device=dev)
    st.order()
    T = {"engine": [], "k1": [], "sort": []}
    for i in range(n_events // batch):
        sl = slice(i * batch, (i + 1) * batch)
        ev_ = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        app = d["app"][sl]
        ev_[0].record()
        st.unit_idx.index_copy_(0, app.long(), d["next"][sl])
        g = st.graph_idx.index_select(0, app.long())
        eng.run(g, d["next"][sl], d["seed"][sl], d["comp"][sl], d["obs"][sl], n=512,
                bucket_count=256, queue=hq, slots=app)
        ev_[1].record()
        hq.est_age.index_copy_(0, app.long(), att[sl])
        hq.age.index_copy_(0, app.long(), att[sl])
        hq.score(2.0, rows=app)
        ev_[2].record()
        st._update_order(app)
        ev_[3].record()
        torch.cuda.synchronize()
        if i >= 2:
            T["engine"].append(ev_[0].elapsed_time(ev_[1]))
            T["k1"].append(ev_[1].elapsed_time(ev_[2]))
            T["sort"].append(ev_[2].elapsed_time(ev_[3]))
    print(json.dumps({"full_queue_engine_ms_1M_template_apps": full,
                      **{k: float(np.mean(v)) for k, v in T.items()}}))


if __name__ == "__main__":
    main()
