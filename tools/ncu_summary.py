"""Summarise ncu reports of the SSA kernels into JSON (for profiles/).

    python tools/ncu_summary.py OUT.json name=report.ncu-rep [name=report.ncu-rep ...]

Per report (first profiled kernel): duration, warp instructions, issue-slot
utilisation, SIMT efficiency, warp latency per instruction, occupancy,
fp64-pipe utilisation, divergent branches, the top stall reasons and DRAM
traffic (dram__bytes_read.sum + dram__bytes_write.sum, the `traffic` field
of bench.py's roofline).
"""
import csv
import json
import subprocess
import sys

KEYS = {
    "kernel": "Kernel Name",
    "duration_ms": "gpu__time_duration.sum",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "warp_inst": "smsp__inst_executed.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "threads_per_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
    "warp_latency_per_inst": "smsp__average_warp_latency_per_inst_issued.ratio",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "max_warps_pct": "sm__maximum_warps_per_active_cycle_pct",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "branch_targets": "smsp__sass_branch_targets.sum",
    "branch_targets_divergent": "smsp__sass_branch_targets_threads_divergent.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "sm_clock_hz": "sm__cycles_elapsed.avg.per_second",
}
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "ms": 1.0, "us": 1e-3, "ns": 1e-6, "s": 1e3,
         "Ghz": 1e9, "Mhz": 1e6, "hz": 1.0}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    s = {}
    for k, name in KEYS.items():
        if name not in d:
            continue
        v, u = d[name]
        try:
            x = float(v.replace(",", ""))
            s[k] = x * SCALE.get(u, 1.0)
        except ValueError:
            s[k] = v
    st = []
    for h, (v, u) in d.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                st.append((h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(v)))
            except ValueError:
                pass
    st.sort(key=lambda x: -x[1])
    s["stalls_per_issue"] = dict(st[:8])
    # pipe mix: warp instructions per pipe, as fractions of all executed
    pipes = {}
    for h, (v, u) in d.items():
        if "inst_executed_pipe_" in h and h.endswith(".sum"):  # sm__ or smsp__ prefixed, per the ncu version
            try:
                pipes[h[h.index("inst_executed_pipe_") + len("inst_executed_pipe_"):-len(".sum")]] = float(v.replace(",", ""))
            except ValueError:
                pass
    # per-pipe utilisation (what `--set full` carries): instructions executed on the pipe, % of that pipe's peak
    util = {}
    for h, (v, u) in d.items():
        if h.startswith("sm__inst_executed_pipe_") and h.endswith(".avg.pct_of_peak_sustained_active"):
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            if x >= 0.5:
                util[h[len("sm__inst_executed_pipe_"):-len(".avg.pct_of_peak_sustained_active")]] = round(x, 2)
    if util:
        s["pipe_util_pct"] = dict(sorted(util.items(), key=lambda x: -x[1]))
    if pipes and s.get("warp_inst"):
        s["pipe_mix"] = {k: round(v / s["warp_inst"], 4) for k, v in sorted(pipes.items(), key=lambda x: -x[1]) if v > 0}
    # derived: issue fraction per elapsed cycle, SIMT efficiency, useful issue, divergent branch targets
    for k, name in (("inst_issued", "smsp__inst_issued.sum"), ("smsp_cycles_elapsed", "smsp__cycles_elapsed.sum")):
        if name in d:
            try:
                s[k] = float(d[name][0].replace(",", ""))
            except ValueError:
                pass
    if s.get("inst_issued") and s.get("smsp_cycles_elapsed"):
        s["issue_fraction_elapsed"] = s["inst_issued"] / s["smsp_cycles_elapsed"]
    if isinstance(s.get("threads_per_inst"), float):
        s["simt_efficiency"] = s["threads_per_inst"] / 32.0
        if "issue_fraction_elapsed" in s:
            s["useful_issue"] = s["issue_fraction_elapsed"] * s["simt_efficiency"]
    if s.get("branch_targets") and "branch_targets_divergent" in s:
        s["divergent_branch_target_ratio"] = s["branch_targets_divergent"] / s["branch_targets"]
    if "dram_read_bytes" in s and "dram_write_bytes" in s:
        s["dram_bytes"] = s["dram_read_bytes"] + s["dram_write_bytes"]
    return s


def main():
    res = {}
    for arg in sys.argv[2:]:
        name, rep = arg.split("=", 1)
        res[name] = summarise(rep)
        res[name]["report"] = rep
    with open(sys.argv[1], "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
