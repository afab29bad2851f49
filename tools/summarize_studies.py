"""Markdown summaries of tools/parallelism_study.py and tools/ablation_study.py results.

usage: python tools/summarize_studies.py parallelism gpurun_out/r02/parallelism.json > profiles/r02_parallelism.md
       python tools/summarize_studies.py ablation gpurun_out/r02/ablation.json > profiles/r02_ablation.md"""
import collections
import json
import sys

import numpy as np


def ms(xs):
    xs = [x for x in xs if x is not None]
    if not xs:
        return "n/a"
    if len(xs) == 1:
        return f"{xs[0]:.3f}"
    return f"{np.mean(xs):.3f} ± {np.std(xs, ddof=1):.3f}"


def parallelism(path):
    r = json.load(open(path))
    groups = collections.defaultdict(list)
    for run in r["runs"]:
        groups[(run["batch"], run["robots"], run["steps"])].append(run)
    print(f"# Parallelism / batch-size learning study (P:101-112; {r['iters']} policy updates, seeds per point: "
          f"{r['seeds']})\n")
    print("`python tools/parallelism_study.py --baseline` on one B200: curriculum off, every robot on a random level of "
          "the generated 10 x 20 world, pushes / noise / bootstrapping on, 5 epochs x 4 minibatches. Return = mean "
          "episode return (Table 2 reward summed over an episode) over the last 50 updates; time = wall time of the "
          "updates (CUDA-graph iterations incl. the per-iteration statistics read-back).\n")
    print("| batch | robots | steps / robot | return (mean ± sd) | episode length | time for the updates (s) |")
    print("|---:|---:|---:|---:|---:|---:|")
    for (b, n, t), runs in sorted(groups.items()):
        print(f"| {b} | {n} | {t} | {ms([x['return'] for x in runs])} | {ms([x['length'] for x in runs])} | "
              f"{ms([x['wall_s'] for x in runs])} |")


def ablation(path):
    r = json.load(open(path))
    groups = collections.defaultdict(list)
    for run in r["runs"]:
        groups[(run["bootstrap"], run["curriculum"])].append(run)
    print(f"# Time-out bootstrapping / curriculum ablation, paired seeds (NEXT-1; P:46, P:209, P:221; {r['iters']} "
          "updates)\n")
    print("`python tools/ablation_study.py` on one B200: C3 workload (4096 x 24, rough generated world), the same seeds "
          "(initial parameters, world, environment streams) in every arm. Final return = mean episode return over the "
          "last 50 updates; value loss = mean critic loss over the same updates; time-outs = episodes that reached the "
          "1000-step limit in the sampled rollouts (every 25th iteration) -- the only input of the bootstrap.\n")
    print("| bootstrap | curriculum | final return | final value loss | time-outs (sampled rollouts) | mean level (last sample) |")
    print("|---|---|---:|---:|---:|---:|")
    for (bo, cu), runs in sorted(groups.items(), reverse=True):
        print(f"| {bo} | {cu} | {ms([x['final_return'] for x in runs])} | {ms([x['final_value_loss'] for x in runs])} | "
              f"{sum(sum(x['timeouts_every_25']) for x in runs)} | {ms([x['mean_level_every_25'][-1] for x in runs])} |")
    # paired differences
    by = {(x["bootstrap"], x["curriculum"], x["seed"]): x for x in r["runs"]}
    for cu in (True, False):
        d = [by[(True, cu, s)]["final_return"] - by[(False, cu, s)]["final_return"]
             for s in sorted({x["seed"] for x in r["runs"]}) if (True, cu, s) in by and (False, cu, s) in by]
        same = [by[(True, cu, s)]["curves_every_10"] == by[(False, cu, s)]["curves_every_10"]
                for s in sorted({x["seed"] for x in r["runs"]}) if (True, cu, s) in by and (False, cu, s) in by]
        print(f"\ncurriculum {cu}: bootstrap on - off (paired by seed) final return {ms(d)}; identical learning "
              f"curves in {sum(same)} of {len(same)} seeds")


if __name__ == "__main__":
    {"parallelism": parallelism, "ablation": ablation}[sys.argv[1]](sys.argv[2])
