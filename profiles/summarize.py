"""Summarise an ncu launch list and full capture into committed JSON.

    python profiles/summarize.py gpurun_out/launches.csv gpurun_out/prof_full.ncu-rep profiles/r02l [config]

Writes <dir>/launch_shares.json (per-kernel share of the device time of the
steady-state launches: the setup kernels -- graph generator, partition sort,
store init -- are excluded), <dir>/ncu_full_summary.json (per-kernel DRAM
bytes, duration, pipe utilisation, stall reasons) and the config's entry of
profiles/ncu_traffic.json (DRAM bytes per launch for the bench's roofline
`traffic` field; config defaults to tw).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

SETUP = ("powerlaw", "bucket_keys", "gather3", "init_uniform", "DeviceRadixSortHistogram",
         "DeviceRadixSortExclusiveSum")


def short(name):
    n = name.split("(")[0]
    for tag in ("score_kernel", "segment_heads", "long_chunks", "long_combine", "long_index",
                "segment_ws", "segment_flat", "presort_keys", "DeviceSelect",
                "segment_pass1_vec", "segment_pass1", "segment_pass2",
                "loss_reduce", "draw_const", "shuffle_draw", "keys_kernel", "head_kernel",
                "chase_kernel", "final_kernel", "gather_edges", "Onesweep", "Histogram",
                "ExclusiveSum", "zero_kernel", "init_uniform", "powerlaw", "bucket_keys",
                "gather3", "eval_"):
        if tag in n:
            return tag
    return n[-40:]


def launch_shares(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rdr = csv.reader(lines)
    hdr = next(rdr)
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"))
    for r in rdr:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        ms = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0,
              "ms": 1.0}.get(unit, 1e-6) * v
        rows.append((r[ki], ms))
    # steady state: drop everything before the first score_kernel launch
    first = next((i for i, (n, _) in enumerate(rows) if "score_kernel" in n), 0)
    steady = rows[first:]
    tot = sum(ms for _, ms in steady)
    agg = defaultdict(lambda: [0, 0.0])
    for n, ms in steady:
        agg[short(n)][0] += 1
        agg[short(n)][1] += ms
    out = {k: {"launches": c, "ms": round(ms, 4), "share": round(ms / tot, 4)}
           for k, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1])}
    return {"total_launches": len(steady), "total_ms": round(tot, 3), "kernels": out}


def full_summary(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
    stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
             and h.endswith("_per_issue_active.ratio")]
    out = []
    for r in rows[2:]:
        e = {"kernel": r[hdr.index("Kernel Name")]}
        for w in want:
            if w in hdr:
                i = hdr.index(w)
                e[w] = f"{r[i]} {units[i]}".strip()
        st = sorted(((float(r[i]) if r[i] not in ("", "n/a") else 0.0,
                      hdr[i][len("smsp__average_warps_issue_stalled_"):-len(
                          "_per_issue_active.ratio")]) for i in stall), reverse=True)[:5]
        e["top_stalls"] = [[n, round(v, 2)] for v, n in st]
        out.append(e)
    return out


def to_bytes(s):
    v, u = s.split()[0], s.split()[1] if len(s.split()) > 1 else "byte"
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


def main():
    launches, rep, outdir = sys.argv[1], sys.argv[2], sys.argv[3]
    config = sys.argv[4] if len(sys.argv) > 4 else "tw"
    os.makedirs(outdir, exist_ok=True)
    if os.path.exists(launches):
        with open(os.path.join(outdir, "launch_shares.json"), "w") as f:
            json.dump(launch_shares(launches), f, indent=1)
    if os.path.exists(rep):
        full = full_summary(rep)
        with open(os.path.join(outdir, f"ncu_full_summary_{config}.json"), "w") as f:
            json.dump(full, f, indent=1)
        traffic = {}
        def node_pass(name):  # segment_pass1_vec<KIND, NV, REL, SH>: REL == 0
            if "<" not in name:
                return True
            args = [x.strip() for x in name.split("<", 1)[1].split(">")[0].split(",")]
            return len(args) < 3 or args[2] in ("0", "(bool)0", "false")

        for cls, tag in (("score", "score_kernel"), ("update", "segment_heads")):
            hits = [e for e in full if tag in e["kernel"] and node_pass(e["kernel"])]
            if not hits and cls == "update":  # the chunked kernels (LGD_K4=1)
                hits = [e for e in full if "segment_pass1" in e["kernel"] and node_pass(e["kernel"])]
            if hits:
                b = [to_bytes(e["dram__bytes_read.sum"]) + to_bytes(e["dram__bytes_write.sum"])
                     for e in hits]
                traffic[cls] = sum(b) / len(b)
        traffic["source"] = os.path.relpath(
            os.path.join(outdir, f"ncu_full_summary_{config}.json"),
            os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_traffic.json")
        try:
            with open(tpath) as f:
                allt = json.load(f)
        except Exception:
            allt = {}
        allt[config] = traffic
        with open(tpath, "w") as f:
            json.dump(allt, f, indent=1)
    print("ok")


if __name__ == "__main__":
    main()
