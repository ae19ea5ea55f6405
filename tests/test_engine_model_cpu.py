"""The positional stream model behind the GPU engine (tools/engine_model.py)
reproduces the reference Monte Carlo samples (golden hashes) exactly."""

import hashlib

import numpy as np
import pytest

from oracle import pdg_oracle as O
from tools import engine_model as E


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def test_seed_sequence_matches_numpy():
    for seed in [0, 1, 7, 12345, 2**31 - 1, 2**32 + 5, 2**63 + 11, 1000003 * 7 + 3]:
        st = np.random.default_rng(seed).bit_generator.state["state"]
        assert E.seed_state(seed) == (st["state"], st["inc"])


def test_model_reproduces_golden_mc(kb_graphs, mc_cases):
    tables = E.jump_tables(2100)
    gs = {k: O.graph_from_kb(v) for k, v in kb_graphs.items()}
    rejected = 0
    for c in mc_cases["cases"]:
        g = gs[c["graph"]]
        obs = [O.OObs(o["unit_id"], o["input_len"], o["output_len"], o["parallelism"])
               for o in c["obs"]]
        ov = O.conditioning_for(g, c["current"], obs)
        try:
            tot, capped = E.walk(g, c["current"], ov, c["n"], c["seed"], c["visit_cap"], tables)
        except E.Rejected:
            rejected += 1
            continue
        assert _sha(tot) == c["sha256"], c
        assert capped == c["capped"]
    assert rejected <= 2
