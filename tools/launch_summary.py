"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel for one PPO iteration.

usage: python tools/launch_summary.py gpurun_out/launchesN.csv [--md]
The iteration is the span between the 2nd and 3rd k_iter_begin launches (warm-up iterations of bench.py)."""
import collections
import csv
import sys


def main(path, md=False):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    names = [r[4].split("(")[0].replace("void ", "").replace("lg::", "") for r in rows]
    idx = [i for i, n in enumerate(names) if n.startswith("k_iter_begin")]
    a, b = (idx[1], idx[2]) if len(idx) >= 3 else (0, len(rows))
    agg = collections.OrderedDict()
    for r, n in zip(rows[a:b], names[a:b]):
        e = agg.setdefault(n, [0, 0.0])
        e[0] += 1
        e[1] += float(r[-1]) / 1000.0
    tot = sum(v[1] for v in agg.values())
    if md:
        print("| kernel | launches | total us | avg us | share |\n|---|---:|---:|---:|---:|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        if md:
            print(f"| `{k}` | {n} | {t:.1f} | {t / n:.2f} | {100 * t / tot:.1f}% |")
        else:
            print(f"{k:44s} n={n:4d} tot={t:8.1f}us avg={t / n:7.2f}us {100 * t / tot:5.1f}%")
    print(f"\niteration: {b - a} kernels, {tot:.1f} us (serialised, cold-cache ncu durations)")


if __name__ == "__main__":
    main(sys.argv[1], "--md" in sys.argv)
