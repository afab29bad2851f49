"""Deterministic-mean traversability evaluation (§4: "Robots
start in the center of the terrain and are given a forward velocity command of 0.75 m/s, and a side velocity
command randomized within [-0.1, 0.1] m/s" (Fig. traversability caption); "we command the robots to traverse the
representative difficulty of the terrain at high forward velocity and measure the success rate. A success is
defined as managing to cross the terrain while avoiding any contacts on the robot's base").

World: `lg_terrain_generate` (GPU) with L levels x 5 columns, one column per terrain kind
(flat, slope pyramid, rough, obstacles, stairs pyramid), difficulty rising with the level. E robots per tile
spawn at its centre (env_reset with their level / column set), get the command (0.75, U[-0.1, 0.1], 0) m/s, m/s,
rad/s (heading frame; the lateral draw is a seeded host input, tools-side) and run the deterministic policy a = mu
(LG_F_DETERMINISTIC) with no noise, pushes or curriculum. Per robot the first outcome counts: success = its
tile-exit latch (`crossed`, DESIGN.md §3.4 word 64) set before any base contact; failure = a crash (terminated)
first, or neither within --steps policy steps. The success rate is reported per terrain kind and level. Every
step runs in libleggedrl's kernels through the C ABI; this script only reads flags and state words back.
`tests/test_gpu_parity.py::test_traversability_evaluation_vs_oracle` replays the same protocol on the oracle
environment (teacher-forced with the GPU's actions) and checks every robot's outcome and step.

usage: python tools/evaluate.py [--ckpt TRAIN_CKPT.pt] [--levels 10] [--envs-per-tile 32] [--steps 500]
                                [--velocity 0.75] [--lateral 0.1] [--seed 0] [--out gpurun_out/eval.json]
Without --ckpt the policy is synth.init_params (an untrained baseline)."""
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

KINDS = ["flat", "slope", "rough", "obstacles", "stairs"]
S_CMD, S_LEVEL, S_COL, S_CROSSED = 41, 62, 63, 64  # DESIGN.md §3.4 state words


def lateral_commands(n, lateral, seed):
    """The per-robot side velocity command U[-lateral, lateral], a seeded input of the protocol."""
    return np.random.default_rng(1000 + seed).uniform(-lateral, lateral, n).astype(np.float32)


def setup(L, E, steps, seed, theta=None, scan=(17, 11), hidden=(512, 256, 128), velocity=0.75, lateral=0.1):
    """World, context and spawned robots of the protocol; returns (ctx, hf_numpy, cmd [N][3] fp32)."""
    C = len(KINDS)
    N = L * C * E
    hf = torch.empty((80 * L, 80 * C), device="cuda")
    lg.lg_terrain_generate(hf, L, C, seed)
    torch.cuda.synchronize()
    hf_np = hf.cpu().numpy()
    cfg = Config.make(n_envs=N, n_steps=steps, n_minibatches=4, scan_nx=scan[0], scan_ny=scan[1], hidden=hidden,
                      n_levels=L, n_cols=C, flags=lg.F_DETERMINISTIC, seed=seed)
    ctx = Context(cfg, hf_np)
    ctx.params_set(theta if theta is not None else synth.init_params(cfg.obs_dim, cfg.hidden, seed=seed))
    k = torch.arange(N, device=ctx.device) // E  # tile of robot e: level k // C, column k % C
    ctx.reset()
    ctx.sync()
    sw = ctx.state_words
    sw[S_LEVEL].copy_((k // C).int())
    sw[S_COL].copy_((k % C).int())
    ctx.reset(init=False)  # respawn every robot at the centre of its tile
    ctx.sync()
    cmd = np.zeros((N, 3), np.float32)
    cmd[:, 0] = velocity
    cmd[:, 1] = lateral_commands(N, lateral, seed)
    sw[S_CMD:S_CMD + 3].copy_(torch.from_numpy(np.ascontiguousarray(cmd.T)).to(ctx.device).view(torch.int32))
    ctx.sync()
    return ctx, hf_np, cmd


def run(ctx, steps, record=False):
    """The protocol's policy steps: per robot the first outcome (1 success, -1 crash, 0 neither) and its step;
    with record, the actions of every step (for the oracle replay)."""
    N = ctx.cfg.n_envs
    dev = ctx.device
    sw = ctx.state_words
    term = torch.zeros(N, dtype=torch.uint8, device=dev)
    to = torch.zeros(N, dtype=torch.uint8, device=dev)
    outcome = torch.zeros(N, dtype=torch.int8, device=dev)
    steps_to = torch.full((N,), -1, dtype=torch.int32, device=dev)
    acts = []
    for t in range(steps):
        ctx.policy_act(t)
        if record:
            ctx.sync()
            acts.append(ctx.storage("ACT", extra=(12,))[t].cpu().numpy().copy())
        ctx.env_step(t, terminated=term, timeout=to)
        with torch.cuda.stream(ctx.stream):
            crashed = (term != 0) & (outcome == 0)
            crossed = (sw[S_CROSSED] != 0) & (outcome == 0) & ~crashed
            outcome.masked_fill_(crashed, -1)
            outcome.masked_fill_(crossed, 1)
            steps_to.masked_fill_(crashed | crossed, t + 1)
    ctx.sync()
    return outcome.cpu().numpy(), steps_to.cpu().numpy(), acts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ckpt", default=None, help="checkpoint of tools/train.py (its policy weights are used)")
    ap.add_argument("--levels", type=int, default=10)
    ap.add_argument("--envs-per-tile", type=int, default=32)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--velocity", type=float, default=0.75)
    ap.add_argument("--lateral", type=float, default=0.1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "eval.json"))
    args = ap.parse_args()
    torch.cuda.set_device(0)
    L, C, E = args.levels, len(KINDS), args.envs_per_tile
    scan, hidden, theta = (17, 11), (512, 256, 128), None
    if args.ckpt:
        ck = torch.load(args.ckpt, weights_only=False)
        scan = (ck["config"]["scan_nx"], ck["config"]["scan_ny"])
        hidden = tuple(ck["config"]["hidden"])
        P = lg.lg_num_params(Config.make(hidden=hidden, scan_nx=scan[0], scan_ny=scan[1]).to_c())
        theta = ck["buffers"][lg.BUF["THETA"]].view(torch.float32)[:P].numpy().copy()
    ctx, _, _ = setup(L, E, args.steps, args.seed, theta, scan, hidden, args.velocity, args.lateral)
    out, stp, _ = run(ctx, args.steps)
    oc = out.reshape(L, C, E)
    st = stp.reshape(L, C, E)
    res = {"levels": L, "envs_per_tile": E, "steps": args.steps, "velocity": args.velocity, "lateral": args.lateral,
           "policy": args.ckpt or "untrained (synth.init_params)", "success": {}, "crash": {}, "mean_steps_to_cross": {}}
    for c, name in enumerate(KINDS):
        res["success"][name] = [float((oc[l, c] == 1).mean()) for l in range(L)]
        res["crash"][name] = [float((oc[l, c] == -1).mean()) for l in range(L)]
        res["mean_steps_to_cross"][name] = [float(st[l, c][oc[l, c] == 1].mean()) if (oc[l, c] == 1).any()
                                            else None for l in range(L)]
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)
    print("success rate per terrain kind (levels 0..L-1):")
    for name in KINDS:
        print(f"  {name:9s} " + " ".join(f"{x:4.2f}" for x in res["success"][name]) +
              "   crash " + " ".join(f"{x:4.2f}" for x in res["crash"][name]))
    ctx.close()


if __name__ == "__main__":
    main()
