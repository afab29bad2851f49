"""Batch-shape sweep (BASELINE.json configs[4]; the throughput side of the paper's
parallelism study, §4.1): N envs x T steps/env x K_mb minibatches, E = 5 epochs, on
the C3 world (rough terrain, 187-point scan, curriculum, noise, pushes), one B200.

Per point: CUDA-graph replay of the full iteration (rollout + GAE + E*K_mb minibatch updates), L2 flushed
before every timed iteration, CUDA events on the library stream, median of --iters after 3 warm-ups;
one profiled replay for the GEMM share; one lg_iterate_host call whose stats must report E*K_mb applied
minibatches and no non-finite skips (sanity, not parity: parity is tests/test_gpu_parity.py).

Reported roofline fraction = t_roofline / t_measured with t_roofline = algorithmic FLOPs of the iteration
(bench.algorithmic) at the measured bf16 sustained peak; `gemm_frac` is the same figure for
the GEMM launches alone.

usage: python tools/sweep.py [--quick] [--iters K] [--out gpurun_out/sweep.json]
       python tools/sweep.py --md gpurun_out/sweep.json ROUND > profiles/ROUND_sweep.md"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2109_11978_b200 import lg  # noqa: E402
from paper_2109_11978_b200.context import Config, Context  # noqa: E402

NS = [512, 1024, 2048, 4096, 8192, 16384]
TS = [8, 16, 24, 32, 50]
KS = [1, 2, 4, 8, 16]
PAPER_B = {49152, 98304, 196608}  # P:101 batch sizes


def point(hf, n, t, k, iters, flush, pk):
    w = dict(bench.WORKLOADS["rough"], n_envs=n, n_steps=t)
    cfg = Config.make(n_envs=n, n_steps=t, n_minibatches=k, hidden=w["hidden"], scan_nx=17, scan_ny=11,
                      n_levels=10, n_cols=20, flags=w["flags"], seed=1234)
    ctx = Context(cfg, hf)
    try:
        ctx.params_set(synth.init_params(cfg.obs_dim, cfg.hidden, seed=1234))
        ctx.reset()
        ctx.capture()
        for _ in range(3):
            ctx.replay()
        ctx.sync()
        ms = []
        for _ in range(iters):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(ctx.stream):
                flush.zero_()
                a.record(ctx.stream)
            ctx.replay()
            with torch.cuda.stream(ctx.stream):
                b.record(ctx.stream)
            ctx.sync()
            ms.append(a.elapsed_time(b))
        ctx.profile(True)
        ctx.capture()
        ctx.replay()
        ctx.sync()
        cats = ctx.profile_read()
        ctx.profile(False)
        ctx.capture()
        st = ctx.iterate_host()
        alg = bench.algorithmic(cfg, w)
        med = statistics.median(ms)
        gcat = ["gemm_fwd", "gemm_dw", "gemm_dx", "gemm_roll"]
        gms = sum(cats[c][0] for c in gcat)
        gfl = sum(alg[c] for c in gcat)
        peak = pk["bf16_sus"] * 1e12
        ok = st.minibatches_applied == 5 * k and st.nonfinite_skips == 0
        return dict(n_envs=n, n_steps=t, n_minibatches=k, batch=n * t, minibatch=n * t // k,
                    paper_batch=n * t in PAPER_B, ms_median=med, ms_p10=sorted(ms)[len(ms) // 10],
                    ms_p90=sorted(ms)[min(len(ms) - 1, (9 * len(ms)) // 10)],
                    env_steps_per_s=n * t / (med * 1e-3), tflop_per_iter=alg["total_flops"] / 1e12,
                    roofline_frac=alg["total_flops"] / peak / (med * 1e-3),
                    gemm_ms=gms, gemm_share=gms / sum(v[0] for v in cats.values()),
                    gemm_frac=gfl / peak / (gms * 1e-3) if gms else None,
                    phase_ms={c: round(v[0], 4) for c, v in cats.items() if v[1]}, sane=bool(ok))
    finally:
        ctx.close()
        del ctx
        torch.cuda.empty_cache()


def render(path, rnd):
    d = json.load(open(path))
    pts = {(r["n_envs"], r["n_steps"], r["n_minibatches"]): r for r in d["points"]}
    print(f"# {rnd}: batch-shape sweep (BASELINE configs[4], SURVEY C5), one B200\n")
    print("`tools/sweep.py`: C3 world (rough terrain, 187-point scan, curriculum, noise, pushes), MLP 512-256-128, "
          f"E = 5 epochs; per point the median of {d['iters']} graph replays of the whole iteration (L2 flushed, CUDA "
          "events). Roofline fraction = algorithmic FLOPs of the iteration at the measured bf16 sustained peak "
          f"({d['peaks']['bf16_sus']:.0f} TFLOP/s) / measured time; GEMM fraction = the same for the GEMM launches "
          "alone (profiled replay). Every point passed the sanity check (E*K_mb minibatches applied, no "
          "non-finite skips). **Bold**: the paper's batch sizes B in {49152, 98304, 196608} (P:101).\n")
    for k in KS:
        print(f"\n## K_mb = {k} minibatches: ms / iteration (M env-steps/s, roofline fraction, GEMM fraction)\n")
        print("| N envs \\ T steps | " + " | ".join(str(t) for t in TS) + " |")
        print("|---|" + "---:|" * len(TS))
        for n in NS:
            cells = []
            for t in TS:
                r = pts.get((n, t, k))
                if not r:
                    cells.append("")
                    continue
                c = (f"{r['ms_median']:.2f} ({r['env_steps_per_s'] / 1e6:.1f}, {r['roofline_frac']:.3f}, "
                     f"{(r['gemm_frac'] or 0):.3f})")
                cells.append(f"**{c}**" if r["paper_batch"] else c)
            print(f"| {n} | " + " | ".join(cells) + " |")
    best = max(d["points"], key=lambda r: r["roofline_frac"])
    print(f"\nHighest roofline fraction: {best['roofline_frac']:.3f} at {best['n_envs']} x {best['n_steps']}, "
          f"K_mb = {best['n_minibatches']} ({best['env_steps_per_s'] / 1e6:.1f} M env-steps/s).")


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--md":
        return render(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "r01")
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="N x T on the diagonal-ish subset, K_mb in {1, 4, 16}")
    ap.add_argument("--iters", type=int, default=7)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.json"))
    ap.add_argument("--point", type=int, nargs=3, metavar=("N", "T", "K"), help="one point only (for ncu)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    pk = bench.peaks()
    hf = synth.make_world(10, 20, seed=0, rough=True)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    grid = [(n, t, k) for n in NS for t in TS for k in KS]
    if args.point:
        grid = [tuple(args.point)]
    elif args.quick:
        grid = [(n, t, k) for n in NS for t in (8, 24, 50) for k in (1, 4, 16)]
    res = []
    t0 = time.time()
    for n, t, k in grid:
        r = point(hf, n, t, k, args.iters, flush, pk)
        res.append(r)
        print(json.dumps({x: r[x] for x in ("n_envs", "n_steps", "n_minibatches", "ms_median", "env_steps_per_s",
                                            "roofline_frac", "gemm_frac", "sane")}), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump({"peaks": pk, "iters": args.iters, "wall_s": time.time() - t0, "points": res}, f, indent=1)
    bad = [r for r in res if not r["sane"]]
    print(f"{len(res)} points, {len(bad)} failed sanity, {time.time() - t0:.0f} s")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
