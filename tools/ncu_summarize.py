"""Summarise ncu captures (gpurun_out/*.ncu-rep, launches.csv) into profiles/.

    python tools/ncu_summarize.py <round-tag>

Writes profiles/<tag>_ncu.md (human summary) and updates
profiles/ncu_summary.json (machine summary bench.py reads for `traffic`).
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "l1tex__t_sector_hit_rate.pct",
    "lts__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second",
]


def raw(rep: str) -> dict:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for k, u, v in zip(h, units, vals):
        d[k] = (v, u)
    return d


def num(d, k):
    v, u = d.get(k, ("", ""))
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6,
             "ns": 1e-9, "s": 1.0, "Ghz": 1e9, "Mhz": 1e6, "hz": 1.0}.get(u)
    return x * scale if scale else x


def stalls(d, top=6):
    st = []
    for k, (v, _) in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
            try:
                st.append((float(v), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1.0
    return [(k, round(100 * v / tot, 1)) for v, k in sorted(st, reverse=True)[:top]]


def summarize(rep, kernel, apps):
    d = raw(rep)
    dur = num(d, "gpu__time_duration.sum")
    rd, wr = num(d, "dram__bytes_read.sum"), num(d, "dram__bytes_write.sum")
    inst = num(d, "smsp__inst_executed.sum")
    clk = num(d, "sm__cycles_elapsed.avg.per_second")
    sms = 148
    issue_peak = 4 * sms * (clk or 1.965e9) * dur if dur else None
    name = d.get("Kernel Name", (kernel, ""))[0] or kernel
    out = {"kernel": name.split("(")[0], "report": os.path.basename(rep), "apps_per_launch": apps,
           "duration_s": dur, "dram_bytes_per_launch": (rd or 0) + (wr or 0),
           "dram_read": rd, "dram_write": wr, "warp_instructions": inst,
           "issue_active_frac": (num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active")
                                 or 0) / 100.0,
           "issue_frac_of_peak": (inst / issue_peak) if (inst and issue_peak) else None,
           "stalls_pct": stalls(d)}
    for k in METRICS:
        out[k] = num(d, k)
    if kernel == "engine" and dur and inst:
        # issue floors at 4 warp instructions per SM per cycle: all of the
        # kernel's instructions, and only the PCG64 stream's (the 128-bit LCG
        # step, the XSL-RR output and the Lemire draws, pcg64.cuh) -- the
        # part no bookkeeping change can remove
        rate = 4 * sms * (clk or 1.965e9)
        pcg = pcg_instructions(rep)
        out["issue_floor_ms"] = inst / rate * 1e3
        if pcg:
            out["pcg_warp_instructions"] = pcg
            out["pcg_floor_ms"] = pcg / rate * 1e3
    return out


def pcg_instructions(rep):
    """Executed warp instructions attributed to pcg64.cuh source lines."""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    f, tot = None, 0.0
    for r in csv.reader(io.StringIO(txt)):
        if len(r) >= 2 and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if f == "pcg64.cuh" and len(r) > 8 and r[0] not in ("", "Line No"):
            try:
                tot += float(r[7])
            except ValueError:
                pass
    return tot or None


def launches():
    path = os.path.join(OUT, "launches.csv")
    if not os.path.exists(path):
        return []
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    if not rows:
        return []
    h = rows[0]
    try:
        kn, mv, mu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    except ValueError:
        return []
    agg = {}
    for r in rows[1:]:
        try:
            v = float(r[mv].replace(",", ""))
        except ValueError:
            continue
        scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6,
                 "ms": 1e-3}.get(r[mu], 1e-9)
        name = r[kn][:90]
        a = agg.setdefault(name, [0, 0.0, []])
        a[0] += 1
        a[1] += v * scale
        a[2].append(v * scale)
    tot = sum(t for _, t, _ in agg.values()) or 1.0
    MED.clear()
    MED.update({k: sorted(x)[len(x) // 2] for k, (_, _, x) in agg.items()})
    return sorted([(k, n, t, t / tot) for k, (n, t, _) in agg.items()], key=lambda x: -x[2])


MED = {}   # kernel -> median launch time (the bench also runs 1M-app config-3 steps)


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    apps = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
    k1_rows = int(sys.argv[3]) if len(sys.argv) > 3 else 1_000_000   # K1b capture: 1M rows
    os.makedirs(PROF, exist_ok=True)
    js_path = os.path.join(PROF, "ncu_summary.json")
    summ = json.load(open(js_path)) if os.path.exists(js_path) else {}
    lines = [f"# ncu summary ({tag})", ""]
    # role -> report; bench.py reads the "engine" entry for roofline.traffic
    for rep, role, n in (("engine.ncu-rep", "engine", apps), ("k1.ncu-rep", "k1", k1_rows),
                         ("need.ncu-rep", "need", 1_000_000)):
        p = os.path.join(OUT, rep)
        if not os.path.exists(p):
            continue
        s = summarize(p, role, n)
        summ[role] = s
        lines += [f"## {role}: {s['kernel']} (`ncu --set full`, one launch, {n} apps)", "",
                  "| metric | value |", "|---|---|"]
        for k, v in s.items():
            if k in ("kernel", "report"):
                continue
            lines.append(f"| {k} | {v} |")
        lines.append("")
    ls = launches()
    if ls:
        lines += ["## launch list (`ncu --metrics gpu__time_duration.sum`, cold, serialised)",
                  "", "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for k, n, t, f in ls:
            lines.append(f"| `{k}` | {n} | {t * 1e3:.3f} | {f * 100:.1f}% |")
        # the step's own kernels (engine, serial completion, K1, the radix
        # sort of K5): per-launch means, and the engine's share of their sum
        step = [(k, n, t) for k, n, t, _ in ls
                if any(x in k for x in ("mc_walk", "mc_engine", "mc_serial", "gittins_pair",
                                        "gittins_hist", "order_sort", "attained"))]
        if step:
            per = {}
            for k, n, _ in step:
                t = MED[k] * n            # median launch: config-3's 1M-app steps excluded
                grp = ("careful" if "mc_walk" in k and ", 1>" in k else
                       "engine" if ("mc_walk" in k or "mc_engine" in k) else
                       "serial" if "mc_serial" in k else
                       "k1" if "gittins" in k else
                       "attained" if "attained" in k else "sort")
                per.setdefault(grp, [0.0, 0])
                per[grp][0] += t
                # one launch per step per kernel (the unfused attained service
                # is three kernels per step)
                per[grp][1] += n if (grp != "attained" or "fused" in k) else n / 3
            mean = {g: t / max(n, 1) for g, (t, n) in per.items()}
            tot = sum(mean.values()) or 1.0
            summ["launch_step_share"] = {g: m / tot for g, m in mean.items()}
            lines += ["", "Step kernels, mean time per step (cold): " +
                      ", ".join(f"{g} {m * 1e3:.3f} ms" for g, m in mean.items()) +
                      f"; engine share {mean.get('engine', 0.0) / tot * 100:.1f}% "
                      "(bench.py's live share_of_step must agree; per-kernel medians, so "
                      "the 1M-app config-3 launches in the same run do not count)"]
    summ["_tag"] = tag
    json.dump(summ, open(js_path, "w"), indent=1)
    open(os.path.join(PROF, f"{tag}_ncu.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
