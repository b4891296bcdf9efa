"""Summarise ncu reports (raw page) into one JSON per kernel + profiles/ncu_traffic.json.
usage: python scripts/ncu_summary.py <tag>=<report.ncu-rep> ...  > profiles/rNN_ncu_summary.json"""
import csv, io, json, os, subprocess, sys

TRAFFIC = os.environ.get("NCU_TRAFFIC", "profiles/r02_ncu_traffic.json")   # per-config DRAM bytes per launch (bench.py roofline.traffic)

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "launch__registers_per_thread": "registers",
    "launch__block_size": "block",
    "launch__grid_size": "grid",
    "sm__warps_active.avg.per_cycle_active": "warps_active_per_sm",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed": "l1_wavefronts_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__inst_executed_pipe_tma.sum": "tma_inst",
}
STALLS = ["long_scoreboard", "wait", "short_scoreboard", "barrier", "mio_throttle", "selected", "math_pipe_throttle",
          "not_selected", "lg_throttle", "no_instruction", "branch_resolving", "dispatch_stall"]


def raw(rep):
    """A .ncu-rep (read with ncu) or the CSV of its raw page (exported on the GPU box)."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return dict(zip(r[0], r[1])), dict(zip(r[0], r[2]))


res, traffic = {}, {}
for arg in sys.argv[1:]:
    tag, rep = arg.split("=", 1)
    units, d = raw(rep)
    o = {"kernel": d.get("Kernel Name", "")[:90]}
    for k, nm in KEYS.items():
        v = d.get(k)
        if v in (None, ""):
            continue
        v = float(v.replace(",", ""))
        u = units.get(k, "")
        if nm.startswith("dram_") and u in ("Mbyte", "MB"):
            v *= 1e6
        elif nm.startswith("dram_") and u in ("Gbyte", "GB"):
            v *= 1e9
        elif nm.startswith("dram_") and u in ("Kbyte", "KB"):
            v *= 1e3
        if nm == "duration_us" and u in ("msecond", "ms"):
            v *= 1e3
        if nm == "duration_us" and u in ("nsecond", "ns"):
            v *= 1e-3
        o[nm] = v
    tot = 0.0
    st = {}
    for s in STALLS:
        k = f"smsp__average_warp_latency_issue_stalled_{s}.ratio"
        if k in d and d[k] not in ("", None):
            st[s] = float(d[k])
    o["stall_cycles_per_issue"] = {k: round(v, 2) for k, v in sorted(st.items(), key=lambda x: -x[1])[:6]}
    samp = {}
    for k, v in d.items():                         # sampled stall reasons (share of all samples)
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v not in ("", None):
            try:
                samp[k.split("stalled_")[1]] = float(v.replace(",", ""))
            except ValueError:
                pass
    if samp:
        tot_s = sum(samp.values())
        o["stall_samples_share"] = {k: round(v / tot_s, 3) for k, v in sorted(samp.items(), key=lambda x: -x[1])[:6]}
    if "dram_read" in o and "dram_write" in o:
        o["dram_bytes"] = o["dram_read"] + o["dram_write"]
        traffic[tag] = o["dram_bytes"]
    res[tag] = o
print(json.dumps(res, indent=1))
try:                                             # merge: keep the other kernels' entries
    old = json.load(open(TRAFFIC))
except (OSError, ValueError):
    old = {}
old.update(traffic)
json.dump(old, open(TRAFFIC, "w"), indent=1)
