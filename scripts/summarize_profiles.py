"""Summarise round ncu captures into profiles/ (tracked).

    python scripts/summarize_profiles.py r01 gpurun_out/launches_r01_v4.csv gpurun_out/r01_*.ncu-rep
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:   # the driver-measured copy bandwidth of this pool's B200s
    PEAK = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except (OSError, KeyError, ValueError):
    PEAK = 6537.3


def page(rep, name):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv"], capture_output=True,
                         text=True).stdout
    return list(csv.reader(out.splitlines()))


def summarize(rep):
    raw = page(rep, "raw")
    h, units, vals = raw[0], raw[1], raw[2]
    d = dict(zip(h, vals))
    det = page(rep, "details")
    dh = det[0]
    m = {}
    for row in det[1:]:
        r = dict(zip(dh, row))
        m[r["Metric Name"]] = r["Metric Value"]
    f = lambda k: float(d[k].replace(",", "")) if k in d and d[k] not in ("", "n/a") else None
    dur_ns = f("gpu__time_duration.sum")
    rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
    # raw byte metrics are reported in the unit of row 1
    def scale(k):
        u = units[h.index(k)] if k in h else "byte"
        return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    rd *= scale("dram__bytes_read.sum")
    wr *= scale("dram__bytes_write.sum")
    dur_s = dur_ns * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(
        units[h.index("gpu__time_duration.sum")], 1e-9)
    return {
        "report": os.path.basename(rep),
        "kernel": d.get("Kernel Name", "")[:80],
        "duration_us": round(dur_s * 1e6, 2),
        "dram_bytes_read": int(rd), "dram_bytes_write": int(wr),
        "dram_bytes_per_launch": int(rd + wr),
        "dram_GBps": round((rd + wr) / dur_s / 1e9, 1),
        "dram_frac_of_measured_peak": round((rd + wr) / dur_s / 1e9 / PEAK, 4),
        "dram_throughput_pct": m.get("DRAM Throughput"),
        "sm_throughput_pct": m.get("Compute (SM) Throughput"),
        "ipc": m.get("Executed Ipc Active"),
        "achieved_occupancy_pct": m.get("Achieved Occupancy"),
        "registers": m.get("Registers Per Thread"),
        "grid": m.get("Grid Size"), "block": m.get("Block Size"),
    }


def launches(path, frames=4):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(list)
    for x in data:
        name = x["Kernel Name"].split("(")[0].replace("wv::<unnamed>::", "").replace("void ", "")
        agg[name].append(float(x["Metric Value"]) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    return [{"kernel": k, "launches": len(v), "us_per_frame": round(sum(v) / frames, 2),
             "share": round(sum(v) / tot, 4)} for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))]


def main():
    tag, lst, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    out = {"launches": launches(lst), "kernels": [summarize(r) for r in reps]}
    with open(os.path.join(ROOT, "profiles", f"ncu_summary_{tag}.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    for k in out["kernels"]:
        for name, dst in ((f"{tag}_k3_final.ncu-rep", f"ncu_k3_final_{tag}.json"),
                          (f"{tag}_k3_final_full.ncu-rep", f"ncu_k3_final_full_{tag}.json")):
            if k["report"] == name:
                with open(os.path.join(ROOT, "profiles", dst), "w") as fh:
                    json.dump(k, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
