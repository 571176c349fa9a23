#!/usr/bin/env python3
"""Turn a round's gpurun_out/ captures into committed summaries under profiles/.

  python tools/summarize_profiles.py r01

Reads gpurun_out/{bench,bench_ref,launches,host}_<tag>.* and gpurun_out/prof_<tag>.ncu-rep
(via `ncu -i ... --page raw --csv`) and writes profiles/<tag>_summary.md, <tag>_bench.json,
<tag>_launches.csv and <tag>_traffic.json (per-launch DRAM bytes of each kernel, read by
bench.py for the roofline `traffic` field).
"""
import csv
import io
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads/inst"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp insts"),
]


def kname(s):
    s = s.split("(")[0]
    for tok in ("unnamed>::", "void ", "demb200::", "<unnamed>::"):
        s = s.replace(tok, "")
    return s.split("<")[0].strip()


def to_bytes(val, unit):
    f = float(val)
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return f * mult


def ncu_raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return rows[0], rows[1], rows[2:]


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    lines = [f"# Round {tag[1:]} profile summary (B200, sm_100a)", ""]
    host = os.path.join(OUT, f"host_{tag}.txt")
    if os.path.exists(host):
        lines += ["Host / device:", "```", open(host).read().strip(), "```", ""]
    bench = os.path.join(OUT, f"bench_{tag}.json")
    if os.path.exists(bench):
        b = json.loads(open(bench).read().strip().splitlines()[-1])
        json.dump(b, open(os.path.join(PROF, f"{tag}_bench.json"), "w"), indent=1)
        lines += ["## bench.py (N=1)", "",
                  f"* value **{b['value']:.4g} {b['unit']}**, {b['ms_per_step']:.4f} ms/step, "
                  f"{b['steps']} timed steps, L2 flushed between steps",
                  f"* e2e (C ABI, full state both ways, pinned host buffers, readback overlapping the step) "
                  f"{b['e2e']['value']:.4g} {b['unit']}"
                  + (f"; host-coupled motion exchange (72 B up, 76 B down per particle) {b['e2e_motion']['value']:.4g}"
                     if "e2e_motion" in b else ""),
                  f"* roofline: {b['roofline']['kernel']} {b['roofline']['achieved']:.0f} GB/s = "
                  f"{100 * b['roofline']['frac']:.1f}% of {b['roofline']['peak']} GB/s ({b['roofline']['peak_kind']})",
                  f"* clocks: {b['clocks']}"]
        if "cpu_baseline" in b:
            cb = b["cpu_baseline"]
            lines.append(f"* cpu_baseline ({cb['kind']}, {cb['cores']} threads): {cb['value']:.4g} {cb['unit']} — {cb['sample']}")
        lines += ["", "| kernel | ms (events, L2 flushed) |", "|---|---|"]
        for k, v in b["kernel_ms"].items():
            lines.append(f"| {k} | {v:.4f} |")
        lines.append("")
    refb = os.path.join(OUT, f"bench_ref_{tag}.json")
    if os.path.exists(refb):
        r = json.loads(open(refb).read().strip().splitlines()[-1])
        json.dump(r, open(os.path.join(PROF, f"{tag}_bench_reference.json"), "w"), indent=1)
        lines += [f"Reference arm (`--impl reference`): {r['value']:.4g} {r['unit']}, {r['ms_per_step']:.1f} ms/step, "
                  f"{r['cpu_baseline']['cores']} threads.", ""]
    lcsv = os.path.join(OUT, f"launches_{tag}.csv")
    if os.path.exists(lcsv):
        rows = [r for r in csv.DictReader(l for l in open(lcsv) if not l.startswith("=="))]
        with open(os.path.join(PROF, f"{tag}_launches.csv"), "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["id", "kernel", "grid", "block", "duration_ns"])
            for r in rows:
                w.writerow([r["ID"], kname(r["Kernel Name"]), r["Grid Size"], r["Block Size"], r["Metric Value"]])
        per = {}
        for r in rows:
            per.setdefault(kname(r["Kernel Name"]), []).append(float(r["Metric Value"]))
        tot = sum(statistics.median(v) for k, v in per.items() if k != "k_flush")
        lines += ["## ncu launch list (cold-cache, serialised; compare shares)", "",
                  "| kernel | launches | median ns | share of step |", "|---|---|---|---|"]
        for k, v in sorted(per.items(), key=lambda kv: -statistics.median(kv[1])):
            sh = "" if k == "k_flush" else f"{100 * statistics.median(v) / tot:.1f}%"
            lines.append(f"| {k} | {len(v)} | {statistics.median(v):.0f} | {sh} |")
        lines.append("")
    rep = os.path.join(OUT, f"prof_{tag}.ncu-rep")
    traffic, util = {}, {}
    if os.path.exists(rep):
        hdr, units, rows = ncu_raw(rep)
        idx = {h: i for i, h in enumerate(hdr)}
        lines += ["## ncu --set full (one launch each, step 5 of the bench workload)", "",
                  "| kernel | " + " | ".join(n for _, n in METRICS) + " | top stalls (cycles/issue) |",
                  "|" + "---|" * (len(METRICS) + 2)]
        for r in rows:
            name = kname(r[idx["Kernel Name"]])
            cells = []
            for m, _ in METRICS:
                if m in idx:
                    v, u = r[idx[m]], units[idx[m]]
                    if "bytes" in m:
                        cells.append(f"{to_bytes(v, u) / 1e6:.1f} MB")
                    elif m == "gpu__time_duration.sum":
                        cells.append(f"{float(v):.1f} {u}")
                    else:
                        try:
                            cells.append(f"{float(v):.3g}")
                        except ValueError:
                            cells.append(v)
                else:
                    cells.append("?")
            st = []
            for h, i in idx.items():
                if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                    try:
                        st.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            st.sort(reverse=True)
            lines.append(f"| {name} | " + " | ".join(cells) + " | " + ", ".join(f"{n} {v:.2f}" for v, n in st[:3]) + " |")
            rb = to_bytes(r[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_read.sum"]])
            wb = to_bytes(r[idx["dram__bytes_write.sum"]], units[idx["dram__bytes_write.sum"]])
            traffic[name] = rb + wb

            def num(m):
                try:
                    return float(r[idx[m]])
                except (KeyError, ValueError):
                    return None
            tpi = num("smsp__thread_inst_executed_per_inst_executed.ratio")
            util[name] = {"fp64_pipe_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                          "warp_exec_efficiency": tpi / 32.0 if tpi else None,
                          "dram_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                          "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
                          "l2_hit_pct": num("lts__t_sector_hit_rate.pct")}
        lines.append("")
        lines.append("threads/inst / 32 = warp execution efficiency. DRAM traffic is per launch (cold L2 under replay).")
        json.dump(traffic, open(os.path.join(PROF, f"{tag}_traffic.json"), "w"), indent=1)
        json.dump(util, open(os.path.join(PROF, f"{tag}_kernel_util.json"), "w"), indent=1)
    open(os.path.join(PROF, f"{tag}_summary.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
