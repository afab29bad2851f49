"""Parallelism / batch-size learning study (§4.1, Fig. parallelism):
the total reward of an episode after 1500 policy updates and the training time, for a number of robots from
128 to 16384 at three batch sizes (49152, 98304, 196608 samples: n_steps = B / n_robots), against the
20000 robots x 50 steps (1M samples) baseline, over several seeds.

As in the paper the curriculum is removed ("otherwise a more performant policy sees its task difficulty increase")
and robots train directly on the full range of difficulties: every robot gets a uniform random level of the
GPU-generated world (`lg_terrain_generate`, 10 levels x 20 columns, the five terrain kinds) and keeps it. Pushes,
observation noise and time-out bootstrapping stay on; K = 4 minibatches x 5 epochs (Table 3). Every iteration runs
as one CUDA graph of libleggedrl kernels (`lg_iterate_host`: the iteration's statistics come back to the host).

Reported per configuration (mean and sample standard deviation over the seeds): the mean episode return over
the last 50 updates (`lg_update_stats.mean_episode_return`: the summed Table 2 reward of the episodes that ended
in an iteration), the mean episode length, and the wall time of the 1500 updates on this GPU.

The paper's absolute rewards belong to its ANYmal model, PhysX and trained walking policies; on SPEC's transition
model the policy does not learn to walk under Table 2's reward as written (profiles/r01_training.md), so the study
measures how the configurations shape the same learning problem, not the paper's numbers.

usage: python tools/parallelism_study.py [--iters 1500] [--seeds 3] [--robots 128,256,...] [--batches ...]
                                         [--baseline] [--out gpurun_out/parallelism.json]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2109_11978_b200 import lg  # noqa: E402
from paper_2109_11978_b200.context import Config, Context  # noqa: E402

S_LEVEL = 62  # DESIGN.md §3.4 state word
LEVELS, COLS = 10, 20


def run(n, T, iters, seed, hf):
    cfg = Config.make(n_envs=n, n_steps=T, hidden=(512, 256, 128), scan_nx=17, scan_ny=11, n_levels=LEVELS,
                      n_cols=COLS, flags=lg.F_NOISE | lg.F_PUSH | lg.F_BOOTSTRAP, seed=seed, n_minibatches=4,
                      n_epochs=5)
    ctx = Context(cfg, hf)
    ctx.params_set(synth.init_params(cfg.obs_dim, cfg.hidden, seed=seed))
    ctx.reset()
    ctx.sync()
    lev = np.random.default_rng(7000 + seed).integers(0, LEVELS, n).astype(np.int32)  # seeded input
    ctx.state_words[S_LEVEL].copy_(torch.from_numpy(lev).to(ctx.device))
    ctx.reset(init=False)
    ctx.capture()
    rets, lens, eps = [], [], []
    ctx.sync()
    t0 = time.perf_counter()
    for _ in range(iters):
        s = ctx.iterate_host().as_dict()
        rets.append(s["mean_episode_return"])
        lens.append(s["mean_episode_length"])
        eps.append(s["episodes"])
    wall = time.perf_counter() - t0
    ctx.close()
    tail = slice(max(0, iters - 50), iters)
    w = np.asarray(eps[tail], np.float64)
    r = np.asarray(rets[tail], np.float64)
    ln = np.asarray(lens[tail], np.float64)
    ok = w > 0
    return {"return": float((r[ok] * w[ok]).sum() / w[ok].sum()) if ok.any() else None,
            "length": float((ln[ok] * w[ok]).sum() / w[ok].sum()) if ok.any() else None,
            "wall_s": wall, "curve": [float(x) for x in rets[::25]]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=1500)
    ap.add_argument("--seeds", type=int, default=3)
    ap.add_argument("--robots", default="128,256,512,1024,2048,4096,8192,16384")
    ap.add_argument("--batches", default="49152,98304,196608")
    ap.add_argument("--baseline", action="store_true", help="also 20000 robots x 50 steps (1M samples)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "parallelism.json"))
    args = ap.parse_args()
    torch.cuda.set_device(0)
    hfd = torch.empty((80 * LEVELS, 80 * COLS), device="cuda")
    lg.lg_terrain_generate(hfd, LEVELS, COLS, 11)
    torch.cuda.synchronize()
    hf = hfd.cpu().numpy()
    cfgs = [(n, b // n, b) for b in map(int, args.batches.split(",")) for n in map(int, args.robots.split(","))
            if b % n == 0 and (b // n) % 1 == 0]
    if args.baseline:
        cfgs.append((20000, 50, 1000000))
    res = {"iters": args.iters, "seeds": args.seeds, "levels": LEVELS, "cols": COLS, "runs": []}
    if os.path.exists(args.out):  # resume a partial study
        old = json.load(open(args.out))
        if old.get("iters") == args.iters:
            res["runs"] = old["runs"]
    done = {(r["robots"], r["steps"], r["seed"]) for r in res["runs"]}
    for n, T, b in cfgs:
        for seed in range(args.seeds):
            if (n, T, seed) in done:
                continue
            r = run(n, T, args.iters, seed, hf)
            r.update(robots=n, steps=T, batch=b, seed=seed)
            res["runs"].append(r)
            print(f"robots {n:6d} steps {T:5d} batch {b:7d} seed {seed}: return {r['return']} length {r['length']} "
                  f"wall {r['wall_s']:.1f} s", flush=True)
            os.makedirs(os.path.dirname(args.out), exist_ok=True)
            json.dump(res, open(args.out, "w"))
    print("done", len(res["runs"]), "runs")


if __name__ == "__main__":
    main()
