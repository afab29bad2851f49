"""bench.py -- env-steps/s of one whole PPO iteration (rollout of T policy steps x N envs incl. the
transition, rewards, curriculum, observation + height scan; GAE; E x K minibatch PPO update with Alg. 1
+ Adam) on B200, BASELINE.json's metric.  One process per GPU; for N > 1 launch with torchrun.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload rough|flat|c1]

Prints ONE JSON line on rank 0.  The timed region replays a CUDA graph of the whole iteration; every
timed iteration is bracketed by CUDA events on the library stream and preceded (outside the events) by an
L2 flush; the reported time is the max over ranks.  `--impl reference` times the independent CPU oracle
(oracle/, the slow plain implementation) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # BASELINE.json configs[2]: the full hot path incl. the 187-point scan and the curriculum
    "rough": dict(n_envs=4096, n_steps=24, hidden=(512, 256, 128), scan=(17, 11), levels=10, cols=20, rough=True,
                  flags=15, desc="4096 envs x 24 steps rough terrain, 187-pt height scan (235-dim obs), game-inspired "
                                 "curriculum 10 levels x 20 columns, MLP 512-256-128 ELU, batch 98304, 5 epochs x 4 "
                                 "minibatches (BASELINE configs[2])"),
    # BASELINE.json configs[1]
    "flat": dict(n_envs=4096, n_steps=24, hidden=(512, 256, 128), scan=(0, 0), levels=1, cols=1, rough=False,
                 flags=14, desc="4096 envs x 24 steps flat terrain, 48-dim obs, MLP 512-256-128, batch 98304 "
                                "(BASELINE configs[1])"),
    # BASELINE.json configs[0]
    "c1": dict(n_envs=64, n_steps=24, hidden=(128, 64, 32), scan=(0, 0), levels=1, cols=1, rough=False, flags=14,
               desc="64 envs x 24 steps flat, MLP 128-64-32 (BASELINE configs[0])"),
}
METRIC = "env-steps/sec incl. PPO update (4096 envs x 24 steps) at 1/2/4/8 B200"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return dict(hbm=float(j["hbm_gbs"]), bf16=float(j["bf16_tflops"]), bf16_sus=float(j.get("bf16_tflops_sustained",
                    j["bf16_tflops"])), src="measured (MEASURED_PEAKS.json)")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback (B200_PROFILING.md)")


class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, dev):
        self.dev = dev
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in (self.out or "").strip().splitlines():
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        load = [x for x in sm if x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


CAT_KERNEL = {"gemm_dw": "k_gemm_dw", "gemm_fwd": "k_gemm_tc", "gemm_dx": "k_gemm_tc", "gemm_roll": "k_gemm_tc",
              "env": "k_env_step", "loss": "k_loss_heads"}


def measured_traffic(cat):
    """DRAM bytes per launch of the category's kernel from the newest committed ncu --set full summary
    (profiles/rNN_traffic.json, written by tools/make_profile_summary.py), with its capture date and commit:
    ncu cannot run inside the timed bench, so the number is a dated measurement of the same kernel."""
    import glob
    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r*_traffic.json")))
    for f in reversed(files):
        try:
            d = json.load(open(f))
        except (OSError, ValueError):
            continue
        if d.get("kernel") == CAT_KERNEL.get(cat):
            src = "profiles/" + os.path.basename(f)
            return d["traffic_bytes_per_launch"], {"file": src, "captured": d.get("captured"),
                                                   "commit": d.get("commit"), "how": d.get("cache_control")}
    return None, None


def host_cpu():
    """nproc and the CPU model of the host that runs the oracle."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def algorithmic(cfg, w):
    """Algorithmic FLOPs per iteration by category and bytes of the env kernel."""
    D = 48 + w["scan"][0] * w["scan"][1]
    H0, H1, H2 = w["hidden"]
    N, T = w["n_envs"], w["n_steps"]
    B = N * T
    E = 5
    f_fwd = 2 * 2 * (D * H0 + H0 * H1 + H1 * H2)          # hidden layers, actor + critic, per sample
    f_dx = 2 * 2 * (H0 * H1 + H1 * H2)                     # input gradients of layers 2, 3
    Dp = (D + 7) // 8 * 8
    # bf16 operand bytes per sample that the update GEMMs must read and write (activations H_l and
    # gradients dZ_l of both nets; weights and fp32 partials are not counted)
    b_fwd = 2 * (Dp + 2 * H0 + 2 * H1) + 2 * (2 * H0 + 2 * H1 + 2 * H2)
    b_dx = 2 * (2 * H2 + 2 * H1 + 2 * H1) + 2 * (2 * H1 + 2 * H0 + 2 * H0)
    b_dw = 2 * ((Dp + 2 * H0) + (2 * H0 + 2 * H1) + (2 * H1 + 2 * H2))
    return dict(gemm_roll=T * N * f_fwd + N * f_fwd / 2, gemm_fwd=E * B * f_fwd, gemm_dw=E * B * f_fwd,
                gemm_dx=E * B * f_dx,
                bytes_gemm_fwd=E * B * b_fwd, bytes_gemm_dx=E * B * b_dx, bytes_gemm_dw=E * B * b_dw,
                env_bytes_per_step=N * (66 * 4 * 2 + 48 + (D + 7) // 8 * 8 * 2 + 9 + (216 + 36) * 4),
                total_flops=T * N * f_fwd + N * f_fwd / 2 + E * B * (2 * f_fwd + f_dx))


def run_reference(args, w):
    """Reference arm: the oracle as it stands, single-threaded, on a bounded sample of the workload."""
    import numpy as np
    from threadpoolctl import threadpool_limits

    import oracle
    import synth
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_s = min(w["n_envs"], 128)
    hf = synth.make_world(w["levels"], w["cols"], seed=0, rough=w["rough"])
    D = 48 + w["scan"][0] * w["scan"][1]
    th = synth.init_params(D, w["hidden"], seed=0)
    with threadpool_limits(limits=1):
        tr = oracle.Trainer(n_s, w["n_steps"], hf, w["levels"], w["cols"], th, seed=0, scan=w["scan"],
                            hidden=w["hidden"], flags=w["flags"])
        for _ in range(args.warmup):
            tr.run_iteration()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            tr.run_iteration()
        dt = time.perf_counter() - t0
    v = n_s * w["n_steps"] * args.steps / dt
    sample = f"{n_s} envs x {w['n_steps']} steps per step (full iteration incl. 5x4 minibatch update on that batch)"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "env-steps/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 env / f64 learning",
            "data": "synthetic", "config": {"workload": w["desc"], "sample": sample},
            "cpu_baseline": {"value": v, "unit": "env-steps/s", "cores": 1, "kind": "oracle", "sample": sample,
                             **host_cpu()},
            "e2e": {"value": v, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(w, seconds_target=10.0):
    import numpy as np
    from threadpoolctl import threadpool_limits

    import oracle
    import synth
    n_s = min(w["n_envs"], 256)
    hf = synth.make_world(w["levels"], w["cols"], seed=0, rough=w["rough"])
    D = 48 + w["scan"][0] * w["scan"][1]
    th = synth.init_params(D, w["hidden"], seed=0)
    with threadpool_limits(limits=1):
        tr = oracle.Trainer(n_s, w["n_steps"], hf, w["levels"], w["cols"], th, seed=0, scan=w["scan"],
                            hidden=w["hidden"], flags=w["flags"])
        t0 = time.perf_counter()
        it = 0
        while it == 0 or time.perf_counter() - t0 < seconds_target:  # consecutive iterations, >= seconds_target
            tr.run_iteration()
            it += 1
        dt = time.perf_counter() - t0
    return {"value": it * n_s * w["n_steps"] / dt, "unit": "env-steps/s", "cores": 1, "kind": "oracle", **host_cpu(),
            "sample": f"{it} consecutive full iterations of {n_s} envs x {w['n_steps']} steps (same per-sample work: "
                      f"rollout, GAE, 5x4 minibatch update), single thread, {dt:.1f} s"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="rough", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-iters", type=int, default=3)  # >= 1 (the roofline needs the per-category times)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args, w)

    import torch

    import synth
    from paper_2109_11978_b200 import lg
    from paper_2109_11978_b200.context import Config, Context

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = Config.make(n_envs=w["n_envs"], n_steps=w["n_steps"], hidden=w["hidden"], scan_nx=w["scan"][0],
                      scan_ny=w["scan"][1], n_levels=w["levels"], n_cols=w["cols"], flags=w["flags"], seed=1234,
                      rank=rank, world_size=world)
    hf = synth.make_world(w["levels"], w["cols"], seed=0, rough=w["rough"])
    ctx = Context(cfg, hf)
    theta = synth.init_params(cfg.obs_dim, cfg.hidden, seed=1234)
    ctx.params_set(theta)
    if world == 1 and os.environ.get("LG_NCCL_LOOPBACK") == "1":  # diagnostic: the multi-rank path on one GPU
        st, b = lg.lg_nccl_unique_id()
        lg.check(st, what="lg_nccl_unique_id")
        ctx._ck(lg.lg_set_nccl(ctx.ctx, bytes(b)), "lg_set_nccl")
    if world > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            st, b = lg.lg_nccl_unique_id()
            lg.check(st, what="lg_nccl_unique_id")
            uid.copy_(torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda())
        dist.broadcast(uid, 0)
        ctx._ck(lg.lg_set_nccl(ctx.ctx, bytes(uid.cpu().numpy().tobytes())), "lg_set_nccl")
        ctx._ck(lg.lg_broadcast_params(ctx.ctx), "lg_broadcast_params")
    ctx.reset()
    ctx.capture()
    st, n_kernels = lg.lg_graph_kernel_count(ctx.ctx)
    lg.check(st, ctx.ctx, "kernel count")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        ctx.replay()
    ctx.sync()
    # ---------------- timed region
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            with torch.cuda.stream(ctx.stream):
                flush.zero_()                              # L2 flush (outside the events)
                ev[k][0].record(ctx.stream)
            ctx.replay()
            with torch.cuda.stream(ctx.stream):
                ev[k][1].record(ctx.stream)
        ctx.sync()
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = world * cfg.n_envs * cfg.n_steps / (ms_step / 1e3)
    sc = ctx.scalars()
    # ---------------- per-category device time (profiled graph, same workload, run after the timed region)
    ctx.profile(True)
    ctx.capture()
    cats = {k: [0.0, 0] for k in lg.PROF_CATS}
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    prof_ms = 0.0
    for _ in range(args.profile_iters):
        with torch.cuda.stream(ctx.stream):
            flush.zero_()
            t0.record(ctx.stream)
        ctx.replay()
        with torch.cuda.stream(ctx.stream):
            t1.record(ctx.stream)
        ctx.sync()
        prof_ms += t0.elapsed_time(t1)
        for k, (m, c) in ctx.profile_read().items():
            cats[k][0] += m
            cats[k][1] += c
    ctx.profile(False)
    ctx.capture()
    P = max(1, args.profile_iters)
    per_iter = {k: {"ms": v[0] / P, "launches": v[1] // P} for k, v in cats.items() if v[1]}
    alg = algorithmic(cfg, w)
    pk = peaks()
    gemm_cats = ["gemm_fwd", "gemm_dw", "gemm_dx", "gemm_roll"]
    dom = max(per_iter, key=lambda k: per_iter[k]["ms"])
    gflops = sum(alg[k] for k in gemm_cats)
    gms = sum(per_iter.get(k, {"ms": 0})["ms"] for k in gemm_cats)
    if dom in gemm_cats:
        # the MLP GEMMs are the path's one dense contraction, bound by the tensor cores; achieved =
        # algorithmic FLOPs per launch (per-sample FLOPs x rows, Appendix A.2) / the launch's average duration
        # (CUDA event pairs around every launch on its own stream, profiled graph replay inside this run)
        n_l = max(1, per_iter[dom]["launches"])
        flop_launch = alg[dom] / n_l
        ms_launch = per_iter[dom]["ms"] / n_l
        ach = flop_launch / (ms_launch * 1e-3) / 1e12
        roof = {"bound": "tensor", "kernel": f"tcgen05 GEMM ({dom}: {CAT_KERNEL.get(dom)})", "achieved": ach,
                "peak": pk["bf16_sus"], "unit": "TFLOP/s", "frac": ach / pk["bf16_sus"],
                "peak_src": pk["src"] + " bf16 sustained (kernel timed inside a long step)",
                "algorithmic_flop_per_launch": flop_launch, "launches_per_iter": per_iter[dom]["launches"],
                "avg_launch_us": ms_launch * 1e3,
                "frac_of_burst_peak": ach / pk["bf16"]}
        if "bytes_" + dom in alg:
            # NOT algorithmic (SURVEY §8(d) :851-853): the bf16 activation / gradient operands the unfused
            # layer-by-layer GEMMs store and re-read; kept as a labelled secondary view of the same launches
            gbs = alg["bytes_" + dom] / (per_iter[dom]["ms"] * 1e-3) / 1e9
            roof["activation_bytes_view"] = {"note": "non-algorithmic: stored activations/gradients re-read by the "
                                                     "layer-by-layer update GEMMs", "achieved": gbs, "peak": pk["hbm"],
                                             "unit": "GB/s", "frac": gbs / pk["hbm"],
                                             "bytes_per_iter": alg["bytes_" + dom]}
    else:
        if dom == "env":
            nb = alg["env_bytes_per_step"] * cfg.n_steps
        else:
            nb = None
        ach = (nb / (per_iter[dom]["ms"] * 1e-3) / 1e9) if nb else None
        roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": pk["hbm"], "unit": "GB/s",
                "frac": (ach / pk["hbm"]) if ach else None, "peak_src": pk["src"]}
    roof["traffic"], roof["traffic_src"] = measured_traffic(dom)  # DRAM bytes per launch (dated ncu --set full) or None
    roof["all_gemms"] = {"achieved": gflops / (gms * 1e-3) / 1e12 if gms else None, "unit": "TFLOP/s",
                         "frac": (gflops / (gms * 1e-3) / 1e12) / pk["bf16_sus"] if gms else None}
    roof["step_roofline_ms"] = alg["total_flops"] / (pk["bf16_sus"] * 1e12) * 1e3
    # ---------------- end to end through the public API with host buffers (ctrl block in, stats out)
    for _ in range(2):
        ctx.iterate_host()
    if dist:
        dist.barrier()
    te0 = time.perf_counter()
    for _ in range(args.steps):
        stats = ctx.iterate_host()
    te = time.perf_counter() - te0
    tt = torch.tensor([te], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e = world * cfg.n_envs * cfg.n_steps * args.steps / float(tt.item())
    clocks = clk.summary()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "env-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded procedural terrain, random-init actor-critic, simulated robots)",
            "config": {"workload": w["desc"], "n_envs_per_gpu": cfg.n_envs, "n_steps": cfg.n_steps,
                       "global_batch": world * cfg.n_envs * cfg.n_steps, "minibatch": cfg.n_envs * cfg.n_steps // 4,
                       "epochs": 5, "parallelism": f"dp{world}", "precision": "env fp32 (bit-exact to the oracle), "
                       "MLP bf16 operands / fp32 accumulation (tcgen05), GAE/loss/Adam fp32 with fp64 reductions",
                       "l2": "flushed before every timed iteration (512 MiB memset, outside the events)",
                       "timing": "CUDA graph replay of the whole iteration, CUDA events per iteration on the "
                                 "library stream, max over ranks"},
            "clocks": clocks,
            "e2e": {"value": e2e, "unit": "env-steps/s", "h2d_bytes_per_step": 16,
                    "d2h_bytes_per_step": 120, "path": "lg_iterate_host (16-B control block H2D, lg_update_stats "
                                                       "D2H + stream sync every iteration)"},
            "gpu_launches": n_kernels * args.steps,
            "roofline": roof,
            "phase_ms_per_iter": {k: round(v["ms"], 4) for k, v in per_iter.items()},
            "profiled_iter_ms": prof_ms / P,
            "last_update": {k: (round(v, 6) if isinstance(v, float) else v) for k, v in stats.as_dict().items()},
            "device_scalars": sc,
        }
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(w)
        elif not args.no_cpu_baseline:
            line["cpu_baseline"] = None
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
