"""Write the committed profile summaries of a round from the raw gpurun outputs.

usage: python tools/make_profile_summary.py ROUND BENCH_LOG LAUNCH_CSV FULL_REP
  ROUND       e.g. r01
  BENCH_LOG   output of `python bench.py` (last line = the JSON bench line)
  LAUNCH_CSV  ncu --metrics gpu__time_duration.sum --clock-control none --csv launch list of bench.py
  FULL_REP    ncu --set full capture (.ncu-rep) of the dominant kernel inside bench.py

Outputs (under profiles/): ROUND_bench.json, ROUND_launches.md, ROUND_<kernel>_full.md, ROUND_traffic.json
(bench.py reads the newest *_traffic.json for the roofline `traffic` key)."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    names = [r[4].split("(")[0].replace("void ", "").replace("lg::", "") for r in rows]
    ib = [i for i, n in enumerate(names) if n.startswith("k_iter_begin")]
    a, b = (ib[1], ib[2]) if len(ib) >= 3 else (ib[0], ib[1]) if len(ib) == 2 else (0, len(rows))
    agg = collections.OrderedDict()
    for r, n in zip(rows[a:b], names[a:b]):
        e = agg.setdefault(n, [0, 0.0])
        e[0] += 1
        e[1] += float(r[-1]) / 1000.0
    return agg, b - a


def full(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        e = {"kernel": d["Kernel Name"].split("(")[0].replace("void ", ""), "grid": d["Grid Size"], "block": d["Block Size"]}
        for k in KEYS:
            if k in d and d[k] not in ("", "n/a"):
                v = float(d[k].replace(",", ""))
                e[k] = v * SCALE.get(u.get(k, ""), 1.0)
        out.append(e)
    return out


def main():
    rnd, bench_log, launch_csv, rep = sys.argv[1:5]
    os.makedirs(PROF, exist_ok=True)
    line = [ln for ln in open(bench_log).read().splitlines() if ln.startswith("{")][-1]
    bench = json.loads(line)
    with open(os.path.join(PROF, f"{rnd}_bench.json"), "w") as f:
        json.dump(bench, f, indent=1)
    agg, nk = launches(launch_csv)
    tot = sum(v[1] for v in agg.values())
    with open(os.path.join(PROF, f"{rnd}_launches.md"), "w") as f:
        f.write(f"# {rnd}: ncu launch list of one PPO iteration of `bench.py` (rough 4096x24)\n\n")
        f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` (serialised, cold-cache: compare shares).\n\n")
        f.write("| kernel | launches | total us | avg us | share |\n|---|---:|---:|---:|---:|\n")
        for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"| `{k}` | {n} | {t:.1f} | {t / n:.2f} | {100 * t / tot:.1f}% |\n")
        f.write(f"\n{nk} launches, {tot:.1f} us summed; graph replay of the same iteration (CUDA events, bench.py): "
                f"{bench['ms_per_step'] * 1e3:.1f} us.\n")
    caps = full(rep)
    kname = caps[0]["kernel"].replace("lg::", "").split("<")[0] if caps else "kernel"
    with open(os.path.join(PROF, f"{rnd}_{kname}_full.md"), "w") as f:
        f.write(f"# {rnd}: `ncu --set full --clock-control none` of `{kname}` inside bench.py\n\n")
        f.write("| grid | us | DRAM read MB | DRAM write MB | tensor pipe % (active) | L2 % | DRAM % | warps % | issue % | regs |\n")
        f.write("|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|\n")
        for e in caps:
            f.write(f"| {e['grid']} | {e.get('gpu__time_duration.sum', 0):.1f} | {e.get('dram__bytes_read.sum', 0) / 1e6:.1f} | "
                    f"{e.get('dram__bytes_write.sum', 0) / 1e6:.1f} | "
                    f"{e.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                    f"{e.get('lts__throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                    f"{e.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                    f"{e.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                    f"{e.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                    f"{e.get('launch__registers_per_thread', 0):.0f} |\n")
    traffic = [e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0) for e in caps]
    with open(os.path.join(PROF, f"{rnd}_traffic.json"), "w") as f:
        json.dump({"kernel": kname, "launches": len(caps), "traffic_bytes_per_launch": sum(traffic) / max(1, len(traffic)),
                   "per_launch": traffic, "source": os.path.basename(rep), "cache_control": "ncu default (flush)"}, f,
                  indent=1)
    print("wrote", rnd, kname, len(caps), "captures")


if __name__ == "__main__":
    main()
