"""Training driver on the GPU path (SPEC acceptance 7): runs the PPO loop for
many iterations with a metrics stream (one JSON line per iteration), periodic checkpoints and resume
(lg_resume), and reports the mean per-episode velocity-tracking reward (Table 2 terms 1 and 2)
against SPEC's per-episode maximum of (1 + 0.5)·dt·(20 s / dt) = 30 reward units.

Every step of the PPO loop runs in libleggedrl's kernels (policy_act / env_step_obs_reward /
storage_compute_gae / ppo_update through the C ABI). The per-episode tracking sums are bookkeeping on the
caller side (torch ops on the per-step term breakdown `terms`), as a user's logger would do.

usage: python tools/train.py [--terrain flat|rough] [--envs 1024] [--steps 24] [--iters 1500] [--seed 0]
                             [--no-bootstrap] [--no-curriculum] [--out gpurun_out/train] [--ckpt-every 250]
                             [--resume CKPT.pt] [--stop-after K]"""
import argparse
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2109_11978_b200 import lg  # noqa: E402
from paper_2109_11978_b200.context import Config, Context  # noqa: E402

TRACK_MAX = 30.0


def make(args):
    rough = args.terrain == "rough"
    flags = lg.F_NOISE | lg.F_PUSH
    if not args.no_bootstrap:
        flags |= lg.F_BOOTSTRAP
    if rough and not args.no_curriculum:
        flags |= lg.F_CURRICULUM
    levels, cols = (10, 20) if rough else (1, 1)
    cfg = Config.make(n_envs=args.envs, n_steps=args.steps, hidden=(512, 256, 128),
                      scan_nx=17 if rough else 0, scan_ny=11 if rough else 0, n_levels=levels, n_cols=cols,
                      flags=flags, seed=args.seed)
    hf = synth.make_world(levels, cols, seed=args.seed, rough=rough)
    return cfg, hf


class Trainer:
    def __init__(self, cfg, hf, seed):
        self.cfg = cfg
        self.ctx = Context(cfg, hf)
        self.ctx.params_set(synth.init_params(cfg.obs_dim, cfg.hidden, seed=seed))
        dev = self.ctx.device
        N = cfg.n_envs
        self.terms = torch.zeros(N, 9, device=dev)
        self.term = torch.zeros(N, dtype=torch.uint8, device=dev)
        self.to = torch.zeros(N, dtype=torch.uint8, device=dev)
        self.rew = torch.zeros(N, device=dev)
        self.track = torch.zeros(N, dtype=torch.float64, device=dev)   # running per-episode tracking reward
        self.ret = torch.zeros(N, dtype=torch.float64, device=dev)
        self.stats_dev = torch.zeros(ctypes.sizeof(lg.lg_update_stats), dtype=torch.uint8, device=dev)
        self.iteration = 0

    def reset(self):
        self.ctx.reset()

    def state(self):
        ck = self.ctx.checkpoint()
        ck["trainer"] = {"iteration": self.iteration, "track": self.track.cpu(), "ret": self.ret.cpu()}
        return ck

    def load(self, ck):
        self.ctx.restore(ck)
        self.iteration = ck["trainer"]["iteration"]
        self.track.copy_(ck["trainer"]["track"].to(self.track.device))
        self.ret.copy_(ck["trainer"]["ret"].to(self.ret.device))

    def iterate(self):
        ctx, T = self.ctx, self.cfg.n_steps
        ep_track, ep_ret, ep_n = [], [], []
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(ctx.stream):
            t0.record(ctx.stream)
        for t in range(T):
            ctx.policy_act(t)
            ctx.env_step(t, reward=self.rew, terminated=self.term, timeout=self.to, terms=self.terms)
            with torch.cuda.stream(ctx.stream):
                self.track += (self.terms[:, 0] + self.terms[:, 1]).double()
                self.ret += self.rew.double()
                done = (self.term | self.to).bool()
                ep_track.append((self.track * done).sum())
                ep_ret.append((self.ret * done).sum())
                ep_n.append(done.sum())
                self.track.masked_fill_(done, 0.0)
                self.ret.masked_fill_(done, 0.0)
        ctx.compute_gae()
        ctx.update(self.stats_dev)
        with torch.cuda.stream(ctx.stream):
            t1.record(ctx.stream)
            n = torch.stack(ep_n).sum()
            agg = torch.stack([torch.stack(ep_track).sum(), torch.stack(ep_ret).sum(), n.double()])
        ctx.sync()
        s = lg.lg_update_stats.from_buffer_copy(bytes(self.stats_dev.cpu().numpy().tobytes()))
        self.iteration += 1
        tr, rt, ne = agg.cpu().tolist()
        return {"iteration": self.iteration, "episodes": int(ne),
                "track_per_episode": tr / ne if ne else None, "return_per_episode": rt / ne if ne else None,
                "value_loss": s.value_loss, "surrogate": s.surrogate_loss, "entropy": s.entropy,
                "kl": s.mean_kl, "lr": s.lr, "clip_fraction": s.clip_fraction,
                "nonfinite_skips": s.nonfinite_skips, "applied": s.minibatches_applied,
                "promotions": s.promotions, "demotions": s.demotions,
                "mean_level": (sum(i * c for i, c in enumerate(s.level_hist)) / max(1, sum(s.level_hist))),
                "gpu_ms": t0.elapsed_time(t1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--terrain", default="flat", choices=["flat", "rough"])
    ap.add_argument("--envs", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=24)
    ap.add_argument("--iters", type=int, default=1500)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-bootstrap", action="store_true")
    ap.add_argument("--no-curriculum", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "train"))
    ap.add_argument("--ckpt-every", type=int, default=250)
    ap.add_argument("--resume", default=None)
    ap.add_argument("--stop-after", type=int, default=0, help="stop after this many iterations (resume tests)")
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    torch.cuda.set_device(0)
    cfg, hf = make(args)
    tr = Trainer(cfg, hf, args.seed)
    if args.resume:
        tr.load(torch.load(args.resume, weights_only=False))
    else:
        tr.reset()
    tag = f"{args.terrain}_n{args.envs}_t{args.steps}_s{args.seed}" + ("_noboot" if args.no_bootstrap else "") + \
          ("_nocurr" if args.no_curriculum else "")
    log = open(os.path.join(args.out, f"{tag}.jsonl"), "a")
    w0 = time.time()
    window = []
    done_iters = 0
    while tr.iteration < args.iters:
        m = tr.iterate()
        done_iters += 1
        log.write(json.dumps(m) + "\n")
        if m["track_per_episode"] is not None:
            window.append(m["track_per_episode"])
            window = window[-50:]
        if tr.iteration % 100 == 0 or tr.iteration == args.iters:
            avg = sum(window) / len(window) if window else float("nan")
            print(json.dumps({"iteration": tr.iteration, "track_per_episode_avg50": avg,
                              "fraction_of_max": avg / TRACK_MAX, "value_loss": m["value_loss"], "lr": m["lr"],
                              "wall_s": round(time.time() - w0, 1)}), flush=True)
        if args.ckpt_every and tr.iteration % args.ckpt_every == 0:
            torch.save(tr.state(), os.path.join(args.out, f"{tag}_it{tr.iteration}.pt"))
        if args.stop_after and done_iters >= args.stop_after:
            break
    log.close()
    avg = sum(window) / len(window) if window else float("nan")
    print(json.dumps({"final": True, "tag": tag, "iterations": tr.iteration, "track_per_episode_avg50": avg,
                      "fraction_of_max": avg / TRACK_MAX, "wall_s": round(time.time() - w0, 1)}), flush=True)


if __name__ == "__main__":
    main()
