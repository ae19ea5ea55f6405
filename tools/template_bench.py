"""Engine time per template archetype (development tool): 100k apps of one
reference archetype each, current unit drawn over units with successors."""

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
    from tools import synth
    dev = torch.device("cuda", 0)
    with gzip.open(os.path.join(ROOT, "tests", "golden", "graphs.json.gz"), "rt") as fh:
        docs = json.load(fh)
    out = {}
    n = 100_000
    hq = HistQueue(n, 256)
    for name in bench.STREAM_TEMPLATES:
        graphs = {name: graph_from_kb(docs[name])}
        q = synth.template_queue(graphs, n, seed=41)
        eng = DemandEngine(graphs, device=str(dev))
        gi = torch.from_numpy(q["graph"]).to(dev)
        ui = torch.from_numpy(q["unit"].copy()).to(dev)
        seeds = torch.arange(n, dtype=torch.int64, device=dev) * 1000003
        eng.run(gi, ui, seeds, n=512, bucket_count=256, queue=hq)
        ts = []
        for r in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            eng.run(gi, ui, seeds + r, n=512, bucket_count=256, queue=hq)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        own = [u for u, x in graphs[name].units.items() if x.is_llm and x.masks.output_own_input]
        out[name] = {"ms_per_100k": float(np.mean(ts)), "own_units": own}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
