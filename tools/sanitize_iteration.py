"""PPO iterations through the C ABI with eager launches (no CUDA graph: both streams, cooperative and cluster
launches as issued), for tools that cannot follow a graph replay -- compute-sanitizer, ncu's replay of the
cooperative CTA-pair weight-gradient kernel:
    python tools/sanitize_iteration.py [n_envs T iterations]     (default 256 8 1; C3 = 4096 24)
Exits non-zero if the library reports an error or the update is not finite."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2109_11978_b200.context import Config, Context  # noqa: E402


def main(n_envs=256, T=8, iters=1):
    cfg = Config.make(n_envs=n_envs, n_steps=T, hidden=(512, 256, 128), scan_nx=17, scan_ny=11, n_levels=10, n_cols=20,
                      flags=15, seed=3, n_minibatches=4, n_epochs=5)
    ctx = Context(cfg, synth.make_world(10, 20, seed=3, rough=True))
    ctx.params_set(synth.init_params(cfg.obs_dim, cfg.hidden, seed=3))
    ctx.reset()
    for _ in range(iters):
        ctx.iteration()
    ctx.sync()
    th = ctx.theta.cpu().numpy()
    assert np.all(np.isfinite(th))
    print("sanitize iteration ok", n_envs, T, float(np.abs(th).sum()))


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:4]])
