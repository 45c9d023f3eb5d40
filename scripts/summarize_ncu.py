"""Summarise ncu reports / launch lists into profiles/ (committed evidence).

    python scripts/summarize_ncu.py launches <launches.csv> <out.txt>
    python scripts/summarize_ncu.py full <report.ncu-rep> <out.txt>
"""
import collections
import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr, ks = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            v, u = float(d["Metric Value"]), d["Metric Unit"]
            us = v / 1e3 if u in ("nsecond", "ns") else (v if u in ("usecond", "us") else v * 1e3)
            ks.append((d["Kernel Name"].split("(")[0], us))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, v in ks:
        agg[k][0] += 1
        agg[k][1] += v
    # (with --kernel-name-base demangled ncu prints "void unnamed>::..." for
    # the kernels of libskp's anonymous namespace)
    def mine(k):
        return "skp::" in k or k.startswith("void unnamed>::") or k.startswith("unnamed>::")
    ours = {k: v for k, v in agg.items() if mine(k)}
    tot = sum(v[1] for v in ours.values())
    with open(out, "w") as f:
        f.write(f"# launch list summary of {path}\n# (cold-cache, serialised: compare SHARES)\n")
        f.write(f"# libskp kernels: {sum(v[0] for v in ours.values())} launches, {tot/1e3:.2f} ms\n")
        f.write(f"{'ms':>10} {'share':>6} {'n':>5}  kernel\n")
        for k, v in sorted(ours.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{v[1]/1e3:10.3f} {v[1]/tot*100:5.1f}% {v[0]:5d}  {k}\n")
        other = {k: v for k, v in agg.items() if not mine(k)}
        f.write("# non-libskp kernels (input generation by torch, not in the timed region)\n")
        for k, v in sorted(other.items(), key=lambda kv: -kv[1][1])[:10]:
            f.write(f"{v[1]/1e3:10.3f}        {v[0]:5d}  {k[:100]}\n")


def full(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary of {path}\n")
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            f.write(f"\n## {d.get('Kernel Name', '?')[:120]}\n")
            for k in KEYS:
                if k in d:
                    f.write(f"{k:85s} {units[hdr.index(k)]:8s} {d[k]}\n")


def traffic(out, *reps):
    """profiles/traffic.json: DRAM bytes (read + write) per launch of each
    captured kernel, for bench.py's roofline "traffic" field.
        python scripts/summarize_ncu.py traffic profiles/traffic.json key=report.ncu-rep ..."""
    import json
    res = {}
    for kv in reps:
        key, path = kv.split("=", 1)
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        hdr, units, vals = rows[0], rows[1], rows[2]
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(d[k]) * scale[u[k]]
        res[key] = {"bytes_per_launch": tot, "source": path.split("/")[-1],
                    "kernel": d.get("Kernel Name", "?")[:80]}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(sys.argv[2], *sys.argv[3:])
    else:
        {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
