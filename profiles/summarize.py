#!/usr/bin/env python
"""Summarise the ncu outputs of profiles/run_profiles.sh (copied from gpurun_out/).

    python profiles/summarize.py <dir with launches.csv and full_*.ncu-rep> <round tag>

Writes profiles/<tag>_launches.csv (the per-launch list), profiles/<tag>_summary.md
(per-kernel-family share of the step from the launch list, and the --set full metrics
of one launch per family) and profiles/ncu_traffic.json (DRAM bytes per launch of each
family, read by bench.py for roofline.traffic).
"""
import csv
import io
import json
import os
import re
import shutil
import subprocess
import sys
from collections import defaultdict

HERE = os.path.dirname(os.path.abspath(__file__))
FAMILY = [("k_col_cluster", "col_pass (cluster)"), ("k_col_pass", "col_pass (band tuples)"),
          ("k_row_pass", "row_pass"), ("k_update", "update"), ("k_guide_deriv", "guide_deriv"),
          ("k_prologue", "prologue"), ("k_rank_compose", "rank_compose"), ("k_seam_fix", "seam_fix"),
          ("k_edge_length", "edge_length (create)"), ("k_edge_profiles", "edge_profiles (create)")]
BENCH_NAME = {"k_col_cluster": "col_pass", "k_row_pass": "row_pass", "k_update": "update",
              "k_guide_deriv": "guide_deriv", "k_prologue": "prologue", "k_col_pass": "col_pass",
              "k_seam_fix": "seam_fix"}


def row_mode(name):
    """MODE template argument of a k_row_pass instance (mangled ILi<L>ELi<CT>ELi<MODE>E or
    demangled k_row_pass<L, CT, MODE>)."""
    m = re.search(r"k_row_pass(?:ILi\d+ELi\d+ELi(\d)E|<\s*\d+,\s*\d+,\s*(\d)\s*>)", name)
    return int(m.group(1) or m.group(2)) if m else 0


def family(name):
    if "k_row_pass" in name:
        mode = row_mode(name)
        if mode == 3:
            return "k_row_pass", "row_update (row pass + previous Eq. (3) step)"
        if mode == 2:
            return "k_row_pass", "row_pass (support, create)"
    for key, fam in FAMILY:
        if key in name:
            return key, fam
    return name, name


def read_launches(path):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = defaultdict(lambda: defaultdict(float))
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        try:
            v = float(r[ix["Metric Value"]].replace(",", ""))
        except ValueError:
            continue
        per[(r[ix["ID"]], r[ix["Kernel Name"]])][r[ix["Metric Name"]] + " [" + r[ix["Metric Unit"]] + "]"] = v
    return per


def to_ns(d, key_prefix):
    for k, v in d.items():
        if k.startswith(key_prefix):
            unit = k[k.rfind("[") + 1:-1]
            return v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9}.get(unit, 1)
    return 0.0


def to_bytes(d, key_prefix):
    for k, v in d.items():
        if k.startswith(key_prefix):
            unit = k[k.rfind("[") + 1:-1]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return 0.0


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    hdr, units, vals = rows[0], rows[1], rows[2]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__shared_mem_per_block_dynamic", "launch__cluster_size" if "launch__cluster_size" in hdr else None]
    res = {}
    for h, u, v in zip(hdr, units, vals):
        if h in want:
            res[h] = (v, u)
    return res


def main():
    src = sys.argv[1]
    tag = sys.argv[2]
    launches = os.path.join(src, "launches.csv")
    lines = [f"# ncu summary, {tag}", "",
             "Workload: `python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extras` (C4, 10000x10000, 16-band guide, "
             "20 iterations) on one B200, `--clock-control none`; commands in profiles/run_profiles.sh.", ""]
    traffic = {}
    if os.path.exists(launches):
        shutil.copy(launches, os.path.join(HERE, f"{tag}_launches.csv"))
        per = read_launches(launches)
        fam_t = defaultdict(float)
        fam_n = defaultdict(int)
        fam_b = defaultdict(float)
        for (lid, name), d in per.items():
            key, fam = family(name)
            fam_t[fam] += to_ns(d, "gpu__time_duration.sum")
            fam_n[fam] += 1
            fam_b[fam] += to_bytes(d, "dram__bytes_read.sum") + to_bytes(d, "dram__bytes_write.sum")
        tot = sum(fam_t.values())
        lines += ["## Launch list of one timed step (cold-cache, serialised by ncu: compare SHARES)", "",
                  f"{sum(fam_n.values())} launches, {tot / 1e6:.3f} ms total kernel time.", "",
                  "| family | launches | total ms | share | avg us | DRAM bytes / launch |", "|---|---|---|---|---|---|"]
        for fam in sorted(fam_t, key=lambda f: -fam_t[f]):
            lines.append(f"| {fam} | {fam_n[fam]} | {fam_t[fam] / 1e6:.3f} | {fam_t[fam] / tot:.3f} | "
                         f"{fam_t[fam] / fam_n[fam] / 1e3:.1f} | {fam_b[fam] / fam_n[fam] / 1e6:.1f} MB |")
        lines.append("")
    lines += ["## `--set full`, one launch per family", ""]
    for f in sorted(os.listdir(src)):
        m = re.match(r"full_(\w+)\.ncu-rep", f)
        if not m:
            continue
        key = m.group(1)
        dst = os.path.join(HERE, f"{tag}_{key}.ncu-rep")
        shutil.copy(os.path.join(src, f), dst)
        met = full_metrics(dst)
        if not met:
            continue
        rd = float(met.get("dram__bytes_read.sum", ("0", ""))[0].replace(",", "")) * \
            {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(met.get("dram__bytes_read.sum", ("", "byte"))[1], 1)
        wr = float(met.get("dram__bytes_write.sum", ("0", ""))[0].replace(",", "")) * \
            {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(met.get("dram__bytes_write.sum", ("", "byte"))[1], 1)
        cfg, base = ("C3", key[3:]) if key.startswith("c3_") else ("C4", key)
        traffic.setdefault(cfg, {})[BENCH_NAME.get(base, base)] = {"dram_bytes_per_launch": rd + wr,
                                                                   "source": os.path.basename(dst)}
        lines.append(f"### {key}  (`{os.path.basename(dst)}`)")
        lines.append("")
        for h, (v, u) in met.items():
            lines.append(f"- {h}: {v} {u}")
        lines.append(f"- DRAM traffic per launch: {(rd + wr) / 1e9:.3f} GB")
        lines.append("")
    c3 = os.path.join(src, "c3_launches.csv")
    if os.path.exists(c3):  # C3 batched: create + five one-iteration solves (tools/c3_batch.py)
        shutil.copy(c3, os.path.join(HERE, f"{tag}_c3_launches.csv"))
        per = read_launches(c3)
        fam_t = defaultdict(float)
        fam_n = defaultdict(int)
        fam_b = defaultdict(float)
        for (lid, name), d in per.items():
            key, fam = family(name)
            fam_t[fam] += to_ns(d, "gpu__time_duration.sum")
            fam_n[fam] += 1
            fam_b[fam] += to_bytes(d, "dram__bytes_read.sum") + to_bytes(d, "dram__bytes_write.sum")
        lines += ["## C3 (8 x 3840x2160, C_t = 3, one batched context): launch list", "",
                  "`C3_ITERS=1 python tools/c3_batch.py` (create, then five one-iteration solves), ncu-serialised.", "",
                  "| family | launches | total ms | avg us | DRAM bytes / launch |", "|---|---|---|---|---|"]
        for fam in sorted(fam_t, key=lambda f: -fam_t[f]):
            lines.append(f"| {fam} | {fam_n[fam]} | {fam_t[fam] / 1e6:.3f} | {fam_t[fam] / fam_n[fam] / 1e3:.1f} | "
                         f"{fam_b[fam] / fam_n[fam] / 1e6:.1f} MB |")
        lines.append("")
    c1 = os.path.join(src, "c1_launches.csv")
    if os.path.exists(c1):  # launch-gap breakdown of one eager C1 solve (tools/c1_once.py)
        shutil.copy(c1, os.path.join(HERE, f"{tag}_c1_launches.csv"))
        per = read_launches(c1)
        durs = [to_ns(d, "gpu__time_duration.sum") for d in per.values()]
        fam_t = defaultdict(float)
        fam_n = defaultdict(int)
        for (lid, name), d in per.items():
            key, fam = family(name)
            fam_t[fam] += to_ns(d, "gpu__time_duration.sum")
            fam_n[fam] += 1
        solve_ms = None
        log = os.path.join(src, "c1_once.log")
        if os.path.exists(log):
            for ln in open(log):
                if "c1_eager_solve_ms" in ln:
                    solve_ms = json.loads(ln)["c1_eager_solve_ms"]
        ksum = sum(durs) / 1e6
        lines += ["## C1 eager solve: kernel time against the event-timed solve", "",
                  f"{len(durs)} consecutive launches of the steady solve sequence (ncu, serialised, caches flushed "
                  f"before each launch, so each duration is an upper bound for the L2-resident C1 planes): "
                  f"{ksum:.3f} ms of kernel time.",
                  f"The same solve timed with CUDA events without ncu (programmatic dependent launch): "
                  f"{solve_ms:.3f} ms." if solve_ms else "", "",
                  "| family | launches | total ms | avg us |", "|---|---|---|---|"]
        for fam in sorted(fam_t, key=lambda f: -fam_t[f]):
            lines.append(f"| {fam} | {fam_n[fam]} | {fam_t[fam] / 1e6:.3f} | {fam_t[fam] / fam_n[fam] / 1e3:.1f} |")
        lines.append("")
    with open(os.path.join(HERE, f"{tag}_summary.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    if traffic:
        tp = os.path.join(HERE, "ncu_traffic.json")
        old = json.load(open(tp)) if os.path.exists(tp) else {}
        for k, v in traffic.items():
            old.setdefault(k, {}).update(v)
        json.dump(old, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
