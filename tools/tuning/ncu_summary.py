"""Summarise ncu reports into profiles/ncu_summary_r01.json (per-launch DRAM
traffic, duration, pipe utilisation, stall mix) + the bench launch list."""
import csv, io, json, subprocess, sys
R = sys.argv[1] if len(sys.argv) > 1 else "r01"
WANT = {
    "gpu__time_duration.sum": "duration_ms",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__grid_size": "grid", "launch__block_size": "block",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3, "ms": 1,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1, "second": 1e3}
out = {}
import os
for name, rep in [("dgemm", "dgemm"), ("ttv", "ttv"), ("innerprod", "innerprod"), ("ttm", "ttm"), ("mttkrp", "mttkrp"),
                  ("g1_grouped", "g1")]:
    if not os.path.exists(f"gpurun_out/{R}_{rep}.ncu-rep"):
        continue
    raw = subprocess.run(["ncu", "-i", f"gpurun_out/{R}_{rep}.ncu-rep", "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[-1]
    d = {"kernel": vals[hdr.index("Kernel Name")]}
    for i, h in enumerate(hdr):
        if h in WANT:
            v = float(vals[i].replace(",", ""))
            u = units[i]
            if WANT[h] in ("dram_read", "dram_write"):
                v *= SCALE.get(u, 1)
            if WANT[h] == "duration_ms":
                v *= SCALE.get(u, 1)
            d[WANT[h]] = v
        if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
            try:
                d.setdefault("stalls", {})[h.split("stalled_")[1]] = float(vals[i])
            except ValueError:
                pass
    st = d.pop("stalls", {})
    tot = sum(st.values()) or 1
    d["stall_share_top"] = {k: round(v / tot, 3) for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:5]}
    d["dram_bytes_per_launch"] = d.get("dram_read", 0) + d.get("dram_write", 0)
    out[name] = d
out["_note"] = ("ncu --set full --clock-control none on one bench-size launch (tools/tuning/prof2.py); "
                "cold-cache, serialised replay: compare shares, not absolute times")
json.dump(out, open(f"profiles/ncu_summary_{R}.json", "w"), indent=1)
for k, v in out.items():
    if k.startswith("_"): continue
    print(k, {x: (round(y, 3) if isinstance(y, float) else y) for x, y in v.items() if x not in ("kernel",)})
