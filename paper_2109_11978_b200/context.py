"""Context: PyTorch-owned device memory + stream around one lg_ctx (plumbing only; every step of the
path runs in libleggedrl's kernels).  Config defaults are PAPER.md Table 3 and DESIGN.md §3."""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field, fields

import torch

from . import lg


@dataclass
class Config:
    n_envs: int = 4096
    n_steps: int = 24
    n_epochs: int = 5
    n_minibatches: int = 4
    hidden: tuple = (512, 256, 128)
    scan_nx: int = 17
    scan_ny: int = 11
    n_levels: int = 10
    n_cols: int = 20
    inv_cell: float = 10.0
    gamma: float = 0.99
    lam: float = 0.95
    clip: float = 0.2
    vclip: float = 0.2
    ent_coef: float = 0.01
    vf_coef: float = 1.0
    kl_target: float = 0.01
    lr_init: float = 1e-3
    adam_b1: float = 0.9
    adam_b2: float = 0.999
    adam_eps: float = 1e-8
    seed: int = 0
    rank: int = 0
    world_size: int = 1
    flags: int = lg.F_CURRICULUM | lg.F_NOISE | lg.F_PUSH | lg.F_BOOTSTRAP

    @classmethod
    def make(cls, **kw):
        names = {f.name for f in fields(cls)}
        bad = set(kw) - names
        if bad:  # unknown keys are rejected
            raise ValueError(f"unknown config keys: {sorted(bad)}")
        return cls(**kw)

    def to_c(self) -> lg.lg_config:
        c = lg.lg_config()
        c.struct_size = ctypes.sizeof(lg.lg_config)
        for f in fields(self):
            v = getattr(self, f.name)
            if f.name == "hidden":
                c.hidden = (ctypes.c_int32 * 3)(*v)
            else:
                setattr(c, f.name, v)
        return c

    @property
    def obs_dim(self):
        return 48 + self.scan_nx * self.scan_ny

    @property
    def obs_stride(self):
        return (self.obs_dim + 7) // 8 * 8


class Context:
    def __init__(self, cfg: Config, heightfield, device="cuda", stream=None):
        self.cfg = cfg
        self.c = cfg.to_c()
        st, sizes = lg.lg_required_sizes(self.c)
        lg.check(st, what="lg_required_sizes")
        self.device = torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        torch.cuda.set_device(self.device)
        self.stream = stream if stream is not None else torch.cuda.Stream(device=self.device)
        self.bufs = [torch.empty(max(int(s), 256), dtype=torch.uint8, device=self.device) for s in sizes]
        hf = torch.as_tensor(heightfield, dtype=torch.float32).contiguous()
        assert hf.shape == (80 * cfg.n_levels, 80 * cfg.n_cols), hf.shape
        self.bufs[lg.BUF["HEIGHTFIELD"]][: hf.numel() * 4].copy_(hf.view(-1).view(torch.uint8))
        torch.cuda.synchronize(self.device)
        st, self.ctx = lg.lg_create(self.c, self.bufs, self.stream.cuda_stream)
        lg.check(st, None, "lg_create")
        self.P = int(lg.lg_num_params(self.c))
        self.N, self.T = cfg.n_envs, cfg.n_steps
        self.D, self.Dp = cfg.obs_dim, cfg.obs_stride

    # ---- typed views of the caller-owned buffers ------------------------------------------------
    def view(self, name, dtype, shape):
        b = self.bufs[lg.BUF[name]]
        n = 1
        for s in shape:
            n *= s
        return b[: n * torch.tensor([], dtype=dtype).element_size()].view(dtype).view(*shape)

    @property
    def state_words(self):
        return self.view("STATE", torch.int32, (66, self.N))

    @property
    def obs(self):
        return self.view("OBS", torch.bfloat16, (self.T + 1, self.N, self.Dp))

    def storage(self, name, dtype=torch.float32, extra=()):
        return self.view(name, dtype, (self.T, self.N, *extra))

    @property
    def theta(self):
        return self.view("THETA", torch.float32, (self.P,))

    @property
    def grad(self):
        return self.view("GRAD", torch.float32, (self.P + 16,))

    # ---- calls (marshalling only) ------------------------------------------------------------------
    def _ck(self, st, what):
        lg.check(st, self.ctx, what)

    def _enter(self):
        # order the context stream after work the caller enqueued on the current torch stream
        self.stream.wait_stream(torch.cuda.current_stream(self.device))

    def params_set(self, theta):
        th = torch.as_tensor(theta, dtype=torch.float32).to(self.device).contiguous()
        self._enter()
        self._ck(lg.lg_params_set(self.ctx, th), "lg_params_set")
        self.stream.synchronize()

    def reset(self, mask=None, init=True, obs=None):
        self._enter()
        self._ck(lg.env_reset(self.ctx, mask, int(init), obs), "env_reset")

    def policy_act(self, t, **outs):
        self._enter()
        self._ck(lg.policy_act(self.ctx, t, **outs), "policy_act")

    def env_step(self, t, **kw):
        self._enter()
        self._ck(lg.env_step_obs_reward(self.ctx, t, **kw), "env_step_obs_reward")

    def compute_gae(self, adv=None, ret=None):
        self._enter()
        self._ck(lg.storage_compute_gae(self.ctx, adv, ret), "storage_compute_gae")

    def update(self, stats=None):
        self._ck(lg.ppo_update(self.ctx, stats), "ppo_update")

    def shuffle(self, epoch, perm):
        self._enter()
        self._ck(lg.ppo_shuffle(self.ctx, epoch, perm), "ppo_shuffle")

    def minibatch_grad(self, idx):
        self._enter()
        self._ck(lg.ppo_minibatch_grad(self.ctx, idx, idx.numel()), "ppo_minibatch_grad")

    def forward(self, x_bf16, mu, value):
        self._enter()
        self._ck(lg.policy_forward(self.ctx, x_bf16, x_bf16.shape[0], mu, value), "policy_forward")

    def curriculum(self, crossed, disp, cmd, ep_steps, words, level):
        self._enter()
        self._ck(lg.curriculum_update(self.ctx, level.numel(), crossed, disp, cmd, ep_steps, words, level),
                 "curriculum_update")

    def iteration(self, stats=None):
        for t in range(self.T):
            self.policy_act(t)
            self.env_step(t)
        self.compute_gae()
        self.update(stats)

    def capture(self, stats=None):
        self._ck(lg.lg_graph_capture_iteration(self.ctx, stats), "lg_graph_capture_iteration")

    def replay(self):
        self._ck(lg.lg_graph_launch(self.ctx), "lg_graph_launch")

    def iterate_host(self, ctrl=b"\0" * 16):
        s = lg.lg_update_stats()
        self._ck(lg.lg_iterate_host(self.ctx, ctrl, s), "lg_iterate_host")
        return s

    def scalars(self):
        st, v = lg.lg_device_scalars(self.ctx)
        self._ck(st, "lg_device_scalars")
        import struct
        alpha = struct.unpack("f", struct.pack("i", v[3]))[0]
        kl = struct.unpack("f", struct.pack("i", v[7]))[0]
        return dict(s_base=v[0], iteration=v[1], adam_t=v[2], alpha=alpha, n_to_total=v[4], nonfinite_skips=v[5],
                    applied=v[6], kl_last=kl)

    def adv_normalization(self):
        st, mean, inv_std = lg.lg_adv_normalization(self.ctx)
        self._ck(st, "lg_adv_normalization")
        return mean, inv_std

    def profile(self, enable=True):
        self._ck(lg.lg_profile(self.ctx, enable), "lg_profile")

    def profile_read(self):
        st, ms, cnt = lg.lg_profile_read(self.ctx)
        self._ck(st, "lg_profile_read")
        return {k: (m, c) for k, m, c in zip(lg.PROF_CATS, ms, cnt)}

    def sync(self):
        self.stream.synchronize()

    # ---- checkpoint / resume (lg_resume): all training state is in the caller-owned buffers --------------
    def checkpoint(self):
        """Host copy of every buffer (take it between iterations). Returns {"config": ..., "buffers": [...]}."""
        self.sync()
        return {"config": {f.name: getattr(self.cfg, f.name) for f in fields(self.cfg)},
                "buffers": [b.cpu() for b in self.bufs]}

    def restore(self, ckpt):
        """Load a checkpoint of a context with the same configuration and continue from it."""
        cur = {f.name: getattr(self.cfg, f.name) for f in fields(self.cfg)}
        if {k: (tuple(v) if isinstance(v, (list, tuple)) else v) for k, v in ckpt["config"].items()} != \
                {k: (tuple(v) if isinstance(v, (list, tuple)) else v) for k, v in cur.items()}:
            raise ValueError("checkpoint was taken with a different configuration")
        self.sync()
        for b, h in zip(self.bufs, ckpt["buffers"]):
            if b.numel() != h.numel():
                raise ValueError("checkpoint buffer sizes differ")
            b.copy_(h.to(self.device))
        torch.cuda.synchronize(self.device)
        self._ck(lg.lg_resume(self.ctx), "lg_resume")

    def close(self):
        if getattr(self, "ctx", None):
            lg.lg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Group:
    """All ranks 0..n-1 of one world as contexts on this device (include/lg.h, lg_group_*): the multi-GPU path's
    per-rank work as in one process per GPU, its allreduce as one rank-ordered sum kernel over the ranks' buffers.
    Every context must have been created with world_size = n, its own rank and the same stream."""

    def __init__(self, contexts):
        self.contexts = list(contexts)
        st, self.g = lg.lg_group_create([c.ctx for c in self.contexts])
        self._ck(st, "lg_group_create")

    def _ck(self, st, what):
        if st != 0:
            for c in self.contexts:
                msg = lg.lg_last_error(c.ctx) if c.ctx else ""
                if msg:
                    raise lg.LgError(f"{what}: {lg.STATUS.get(st, st)} {msg}")
            raise lg.LgError(f"{what}: {lg.STATUS.get(st, st)}")

    def broadcast_params(self):
        self._ck(lg.lg_group_broadcast_params(self.g), "lg_group_broadcast_params")

    def compute_gae(self):
        self._ck(lg.lg_group_compute_gae(self.g), "lg_group_compute_gae")

    def update(self, stats=None):
        self._ck(lg.lg_group_ppo_update(self.g, stats), "lg_group_ppo_update")

    def iteration(self, stats=None):
        self._ck(lg.lg_group_iterate(self.g, stats), "lg_group_iterate")

    def sync(self):
        self.contexts[0].sync()

    def close(self):
        if getattr(self, "g", None):
            lg.lg_group_destroy(self.g)
            self.g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
