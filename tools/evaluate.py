"""Deterministic-mean traversability evaluation (§4: "we
command the robots to traverse the representative difficulty of the terrain at high forward velocity and
measure the success rate. A success is defined as managing to cross the terrain while avoiding any contacts
on the robot's base").

World: `lg_terrain_generate` (GPU) with L levels x 5 columns, one column per terrain kind
(flat, slope pyramid, rough, obstacles, stairs pyramid), difficulty rising with the level. E robots per tile
spawn at its centre (env_reset with their level / column set), get the command (v, 0, 0) (forward in their
heading frame; the first observation still carries the command drawn at reset) and run the deterministic
policy a = mu (LG_F_DETERMINISTIC) with no noise, pushes or curriculum. Per robot the first outcome counts:
success = its tile-exit latch (`crossed`, DESIGN.md §3.4 word 64) set before any base contact; failure = a
crash (terminated) first, or neither within --steps policy steps. Every step runs in libleggedrl's kernels
through the C ABI; this script only reads flags and two state words back.

usage: python tools/evaluate.py [--ckpt TRAIN_CKPT.pt] [--levels 10] [--envs-per-tile 32] [--steps 500]
                                [--velocity 1.0] [--seed 0] [--out gpurun_out/eval.json]
Without --ckpt the policy is synth.init_params (an untrained baseline)."""
import argparse
import json
import os
import struct
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2109_11978_b200 import lg  # noqa: E402
from paper_2109_11978_b200.context import Config, Context  # noqa: E402

KINDS = ["flat", "slope", "rough", "obstacles", "stairs"]
S_CMD, S_LEVEL, S_COL, S_CROSSED = 41, 62, 63, 64  # DESIGN.md §3.4 state words


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ckpt", default=None, help="checkpoint of tools/train.py (its policy weights are used)")
    ap.add_argument("--levels", type=int, default=10)
    ap.add_argument("--envs-per-tile", type=int, default=32)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--velocity", type=float, default=1.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "eval.json"))
    args = ap.parse_args()
    torch.cuda.set_device(0)
    L, C, E = args.levels, 5, args.envs_per_tile
    N = L * C * E
    scan = (17, 11)
    theta = None
    if args.ckpt:
        ck = torch.load(args.ckpt, weights_only=False)
        scan = (ck["config"]["scan_nx"], ck["config"]["scan_ny"])
        hidden = tuple(ck["config"]["hidden"])
        P = lg.lg_num_params(Config.make(hidden=hidden, scan_nx=scan[0], scan_ny=scan[1]).to_c())
        theta = ck["buffers"][lg.BUF["THETA"]].view(torch.float32)[:P].numpy().copy()
    hf = torch.empty((80 * L, 80 * C), device="cuda")
    lg.lg_terrain_generate(hf, L, C, args.seed)
    torch.cuda.synchronize()
    cfg = Config.make(n_envs=N, n_steps=args.steps, n_minibatches=4, scan_nx=scan[0], scan_ny=scan[1],
                      n_levels=L, n_cols=C, flags=lg.F_DETERMINISTIC, seed=args.seed)
    ctx = Context(cfg, hf.cpu().numpy())
    ctx.params_set(theta if theta is not None else synth.init_params(cfg.obs_dim, cfg.hidden, seed=args.seed))
    dev = ctx.device
    # tile of robot e: k = e // E, level k // C, column k % C
    k = torch.arange(N, device=dev) // E
    ctx.reset()
    ctx.sync()
    sw = ctx.state_words
    sw[S_LEVEL].copy_((k // C).int())
    sw[S_COL].copy_((k % C).int())
    ctx.reset(init=False)  # respawn every robot at the centre of its tile
    ctx.sync()
    vbits = struct.unpack("<i", struct.pack("<f", args.velocity))[0]
    sw[S_CMD].fill_(vbits)
    sw[S_CMD + 1].zero_()
    sw[S_CMD + 2].zero_()
    term = torch.zeros(N, dtype=torch.uint8, device=dev)
    to = torch.zeros(N, dtype=torch.uint8, device=dev)
    outcome = torch.zeros(N, dtype=torch.int8, device=dev)  # 0 open, 1 success, -1 failure
    steps_to = torch.full((N,), -1, dtype=torch.int32, device=dev)
    for t in range(args.steps):
        ctx.policy_act(t)
        ctx.env_step(t, terminated=term, timeout=to)
        with torch.cuda.stream(ctx.stream):
            crashed = (term != 0) & (outcome == 0)
            crossed = (sw[S_CROSSED] != 0) & (outcome == 0) & ~crashed
            outcome.masked_fill_(crashed, -1)
            outcome.masked_fill_(crossed, 1)
            steps_to.masked_fill_(crashed | crossed, t + 1)
    ctx.sync()
    oc = outcome.view(L, C, E).cpu()
    st = steps_to.view(L, C, E).cpu()
    res = {"levels": L, "envs_per_tile": E, "steps": args.steps, "velocity": args.velocity,
           "policy": args.ckpt or "untrained (synth.init_params)", "success": {}, "crash": {}, "mean_steps_to_cross": {}}
    for c, name in enumerate(KINDS):
        res["success"][name] = [float((oc[l, c] == 1).float().mean()) for l in range(L)]
        res["crash"][name] = [float((oc[l, c] == -1).float().mean()) for l in range(L)]
        res["mean_steps_to_cross"][name] = [float(st[l, c][oc[l, c] == 1].float().mean()) if (oc[l, c] == 1).any()
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
