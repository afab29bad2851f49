"""Time-out bootstrapping and curriculum ablations as paired-seed learning curves (PAPER.md
P:46 "we bootstrap ... on time-outs", P:209 / P:221 App. A.2: bootstrapping "improves the total reward by 10-20 %"
and lowers the critic loss; P:67 the game-inspired curriculum).

Four arms on the C3 workload (4096 robots x 24 steps, rough world of lg_terrain_generate, 10 levels x 20 columns,
pushes and observation noise on): bootstrapping on / off x curriculum on / off, the same seeds in every arm (the
same initial parameters, world and environment random streams: until an episode times out the bootstrap arms are
bit-identical, `test_bootstrap_arms_identical_until_a_timeout`). Per iteration the statistics of `lg_iterate_host`
(mean episode return and length, value loss, surrogate, KL) and, every 25 iterations, the rollout's time-out
count (`n_to_total`, the bootstrap's only input) are recorded.

usage: python tools/ablation_study.py [--iters 1500] [--seeds 3] [--out gpurun_out/ablation.json]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2109_11978_b200 import lg  # noqa: E402
from paper_2109_11978_b200.context import Config, Context  # noqa: E402

LEVELS, COLS = 10, 20


def run(bootstrap, curriculum, seed, iters, hf):
    flags = lg.F_NOISE | lg.F_PUSH | (lg.F_BOOTSTRAP if bootstrap else 0) | (lg.F_CURRICULUM if curriculum else 0)
    cfg = Config.make(n_envs=4096, n_steps=24, hidden=(512, 256, 128), scan_nx=17, scan_ny=11, n_levels=LEVELS,
                      n_cols=COLS, flags=flags, seed=seed)
    ctx = Context(cfg, hf)
    ctx.params_set(synth.init_params(cfg.obs_dim, cfg.hidden, seed=seed))
    ctx.reset()
    ctx.capture()
    keys = ("mean_episode_return", "mean_episode_length", "value_loss", "surrogate_loss", "mean_kl", "episodes")
    hist = {k: [] for k in keys}
    timeouts, levels = [], []
    for it in range(iters):
        s = ctx.iterate_host()
        d = s.as_dict()
        for k in keys:
            hist[k].append(float(d[k]))
        if it % 25 == 0:
            timeouts.append(int(ctx.scalars()["n_to_total"]))
            lh = list(s.level_hist)[:LEVELS]
            levels.append(float(np.dot(lh, np.arange(LEVELS)) / max(1, sum(lh))))
    ctx.close()
    tail = slice(iters - 50, iters)
    w = np.asarray(hist["episodes"][tail], np.float64)
    r = np.asarray(hist["mean_episode_return"][tail], np.float64)
    return {"bootstrap": bootstrap, "curriculum": curriculum, "seed": seed,
            "final_return": float((r * w).sum() / max(w.sum(), 1.0)),
            "final_value_loss": float(np.mean(hist["value_loss"][tail])),
            "timeouts_every_25": timeouts, "mean_level_every_25": levels,
            "curves_every_10": {k: hist[k][::10] for k in keys}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=1500)
    ap.add_argument("--seeds", type=int, default=3)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "ablation.json"))
    args = ap.parse_args()
    torch.cuda.set_device(0)
    hfd = torch.empty((80 * LEVELS, 80 * COLS), device="cuda")
    lg.lg_terrain_generate(hfd, LEVELS, COLS, 11)
    torch.cuda.synchronize()
    hf = hfd.cpu().numpy()
    res = {"iters": args.iters, "runs": []}
    for seed in range(args.seeds):
        for boot in (True, False):
            for cur in (True, False):
                r = run(boot, cur, seed, args.iters, hf)
                res["runs"].append(r)
                print(f"bootstrap {boot!s:5s} curriculum {cur!s:5s} seed {seed}: final return {r['final_return']:.3f} "
                      f"value loss {r['final_value_loss']:.3f} time-outs (per 25 it) {sum(r['timeouts_every_25'])}",
                      flush=True)
                os.makedirs(os.path.dirname(args.out), exist_ok=True)
                json.dump(res, open(args.out, "w"))


if __name__ == "__main__":
    main()
