"""oracle -- TEST INFRASTRUCTURE ONLY.

Independent, plain, slow CPU implementation of the hot path of arXiv 2109.11978:
  * env_oracle.c  -- environment side in fp32 without FMA (Philox, polynomial transcendentals,
                     heightfield lookups, transition, reward, curriculum, reset, observation,
                     Gaussian noise, Feistel shuffle);
  * learn.py      -- learning side in fp64 numpy (MLP fwd/bwd, GAE, PPO loss, Alg. 1, Adam).
It shares no code with paper_2109_11978_b200/ and is only used by tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs.  The product path never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import learn  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "env_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

NW = 66
F_CURRICULUM, F_NOISE, F_PUSH, F_BOOTSTRAP = 1, 2, 4, 8
STATE_DTYPE = np.dtype([
    ("p", "<f4", 3), ("quat", "<f4", 4), ("v", "<f4", 3), ("w", "<f4", 3), ("q", "<f4", 12),
    ("qd", "<f4", 12), ("tair", "<f4", 4), ("cmd", "<f4", 3), ("aprev", "<f4", 12), ("mu", "<f4"),
    ("spawn", "<f4", 2), ("contact", "<u4"), ("push_timer", "<i4"), ("ep_step", "<i4"),
    ("level", "<i4"), ("col", "<i4"), ("crossed", "<u4"), ("ep_return", "<f4")])
assert STATE_DTYPE.itemsize == NW * 4


def build(force: bool = False) -> str:
    """Compile the C oracle: gcc -O2 -ffp-contract=off (no FMA, no fast-math; R26)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Cfg(ctypes.Structure):
    _fields_ = [("n_envs", ctypes.c_int32), ("rank", ctypes.c_int32), ("n_levels", ctypes.c_int32),
                ("n_cols", ctypes.c_int32), ("scan_nx", ctypes.c_int32), ("scan_ny", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("seed_lo", ctypes.c_uint32), ("seed_hi", ctypes.c_uint32),
                ("inv_cell", ctypes.c_float)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        f32p = np.ctypeslib.ndpointer(np.float32, flags="C")
        u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
        _lib.or_philox.argtypes = [ctypes.c_uint32, ctypes.c_uint32, u32p, u32p]
        _lib.or_sincos_batch.argtypes = [ctypes.c_int, f32p, f32p, f32p]
        _lib.or_exp_batch.argtypes = [ctypes.c_int, f32p, f32p]
        _lib.or_log_batch.argtypes = [ctypes.c_int, f32p, f32p]
        _lib.or_h_plate.argtypes = [f32p, ctypes.c_int, ctypes.c_int, ctypes.c_float, ctypes.c_float, ctypes.c_float]
        _lib.or_h_plate.restype = ctypes.c_float
        _lib.or_h_bilinear.argtypes = _lib.or_h_plate.argtypes
        _lib.or_h_bilinear.restype = ctypes.c_float
        _lib.or_curriculum_level.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, ctypes.c_float,
                                             ctypes.c_float, ctypes.c_float, ctypes.c_float, ctypes.c_int32,
                                             ctypes.c_uint32]
        _lib.or_curriculum_level.restype = ctypes.c_int32
        _lib.or_feistel_perm.argtypes = [ctypes.c_uint32, u32p, u32p]
        _lib.or_leg_fk.argtypes = [ctypes.c_int, f32p, ctypes.c_float, f32p, ctypes.c_void_p]
        _lib.or_terrain_generate.argtypes = [f32p, ctypes.c_int, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32]
    return _lib


def terrain_generate(n_levels: int, n_cols: int, seed: int) -> np.ndarray:
    """The world heightfield [80 L][80 C] fp32 of DESIGN.md §3.12 (reading R27)."""
    hf = np.zeros((80 * n_levels, 80 * n_cols), np.float32)
    lib().or_terrain_generate(hf, n_levels, n_cols, seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    return hf


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def philox(k0, k1, ctr):
    out = np.zeros(4, np.uint32)
    lib().or_philox(k0, k1, np.ascontiguousarray(ctr, np.uint32), out)
    return out


def sincos(x):
    x = np.ascontiguousarray(x, np.float32)
    s, c = np.empty_like(x), np.empty_like(x)
    lib().or_sincos_batch(x.size, x, s, c)
    return s, c


def exp(x):
    x = np.ascontiguousarray(x, np.float32)
    y = np.empty_like(x)
    lib().or_exp_batch(x.size, x, y)
    return y


def log(x):
    x = np.ascontiguousarray(x, np.float32)
    y = np.empty_like(x)
    lib().or_log_batch(x.size, x, y)
    return y


def h_plate(hf, x, y, inv_cell=10.0):
    hf = np.ascontiguousarray(hf, np.float32)
    return lib().or_h_plate(hf, hf.shape[0], hf.shape[1], inv_cell, x, y)


def h_bilinear(hf, x, y, inv_cell=10.0):
    hf = np.ascontiguousarray(hf, np.float32)
    return lib().or_h_bilinear(hf, hf.shape[0], hf.shape[1], inv_cell, x, y)


def curriculum_level(level, n_levels, crossed, dx, dy, c0, c1, ep_steps, word):
    return lib().or_curriculum_level(level, n_levels, crossed, dx, dy, c0, c1, ep_steps, word)


def feistel_perm(B, keys):
    perm = np.zeros(B, np.uint32)
    lib().or_feistel_perm(B, np.ascontiguousarray(keys, np.uint32), perm)
    return perm


def leg_fk(leg, q3, knee=False, with_jac=True):
    q3 = np.ascontiguousarray(q3, np.float32)
    pt = np.zeros(3, np.float32)
    J = np.zeros((3, 3), np.float32)
    lsh = np.float32(0.5) * np.float32(0.35) if knee else np.float32(0.35)
    lib().or_leg_fk(leg, q3, float(lsh), pt, J.ctypes.data_as(ctypes.c_void_p) if with_jac else None)
    return pt, J


class Env:
    """Batched environment over the C oracle. State = structured array [N] of STATE_DTYPE."""

    def __init__(self, n_envs, hf, n_levels, n_cols, seed=0, rank=0, scan=(17, 11),
                 flags=F_CURRICULUM | F_NOISE | F_PUSH | F_BOOTSTRAP, inv_cell=10.0):
        self.hf = np.ascontiguousarray(hf, np.float32)
        assert self.hf.shape == (n_levels * 80, n_cols * 80)
        self.cfg = _Cfg(n_envs, rank, n_levels, n_cols, scan[0], scan[1], flags,
                        seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF, inv_cell)
        self.n = n_envs
        self.obs_dim = 48 + scan[0] * scan[1]
        self.state = np.zeros(n_envs, STATE_DTYPE)
        self.s = 0  # env step counter
        L = lib()
        L.or_env_reset.argtypes = [ctypes.POINTER(_Cfg), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p]
        L.or_env_step.argtypes = [ctypes.POINTER(_Cfg), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.or_env_obs.argtypes = [ctypes.POINTER(_Cfg), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32,
                                 ctypes.c_uint32, ctypes.c_void_p]
        L.or_action_eps.argtypes = [ctypes.POINTER(_Cfg), ctypes.c_uint32, ctypes.c_void_p]
        L.or_transition.argtypes = [ctypes.POINTER(_Cfg), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.or_reward_terms.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_float, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]

    def reset(self, mask=None, init=True):
        obs = np.zeros((self.n, self.obs_dim), np.float32)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        lib().or_env_reset(ctypes.byref(self.cfg), _ptr(self.hf), _ptr(self.state), _ptr(m), int(init), self.s,
                           _ptr(obs))
        return obs

    def observe(self, word0=0):
        obs = np.zeros((self.n, self.obs_dim), np.float32)
        lib().or_env_obs(ctypes.byref(self.cfg), _ptr(self.hf), _ptr(self.state), self.s, word0, _ptr(obs))
        return obs

    def step(self, actions):
        self.s += 1
        a = np.ascontiguousarray(actions, np.float32)
        assert a.shape == (self.n, 12)
        obs = np.zeros((self.n, self.obs_dim), np.float32)
        rew = np.zeros(self.n, np.float32)
        term = np.zeros(self.n, np.uint8)
        to = np.zeros(self.n, np.uint8)
        terms = np.zeros((self.n, 9), np.float32)
        tobs = np.zeros((self.n, self.obs_dim), np.float32)
        lib().or_env_step(ctypes.byref(self.cfg), _ptr(self.hf), _ptr(self.state), _ptr(a), self.s, _ptr(obs),
                          _ptr(rew), _ptr(term), _ptr(to), _ptr(terms), _ptr(tobs))
        return obs, rew, term, to, terms, tobs

    def action_eps(self, s=None):
        eps = np.zeros((self.n, 12), np.float32)
        lib().or_action_eps(ctypes.byref(self.cfg), self.s + 1 if s is None else s, _ptr(eps))
        return eps

    def transition_single(self, i, action, s=None):
        """Run only the transition of env i in place; returns tau, qdd, airsum, crash, n_c, and
        the sum of contact normal forces of the last substep."""
        st = self.state[i:i + 1].copy()
        tau = np.zeros(12, np.float32)
        qdd = np.zeros(12, np.float32)
        airsum = ctypes.c_float()
        crash = ctypes.c_int()
        nc = ctypes.c_int()
        fz = ctypes.c_float()
        cfg = _Cfg(1, self.cfg.rank * self.n + i, self.cfg.n_levels, self.cfg.n_cols, self.cfg.scan_nx,
                   self.cfg.scan_ny, self.cfg.flags, self.cfg.seed_lo, self.cfg.seed_hi, self.cfg.inv_cell)
        a = np.ascontiguousarray(action, np.float32)
        lib().or_transition(ctypes.byref(cfg), _ptr(self.hf), _ptr(st), _ptr(a), self.s if s is None else s,
                            _ptr(tau), _ptr(qdd), ctypes.byref(airsum), ctypes.byref(crash), ctypes.byref(nc),
                            ctypes.byref(fz))
        self.state[i] = st[0]
        return tau, qdd, airsum.value, crash.value, nc.value, fz.value


def contact_force(h_ground, pf, vf, mu):
    f = np.zeros(3, np.float32)
    L = lib()
    L.or_contact_force.argtypes = [ctypes.c_float, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_float, ctypes.c_void_p]
    c = L.or_contact_force(h_ground, _ptr(np.ascontiguousarray(pf, np.float32)),
                           _ptr(np.ascontiguousarray(vf, np.float32)), mu, _ptr(f))
    return c, f


def reward_terms(state_rec, action, tau, qdd, airsum, n_c):
    st = np.ascontiguousarray(np.asarray(state_rec, STATE_DTYPE).reshape(1))
    terms = np.zeros(9, np.float32)
    tot = np.zeros(1, np.float32)
    a = np.ascontiguousarray(action, np.float32)
    lib().or_reward_terms(_ptr(st), _ptr(a), _ptr(np.ascontiguousarray(tau, np.float32)),
                          _ptr(np.ascontiguousarray(qdd, np.float32)), ctypes.c_float(airsum), int(n_c),
                          _ptr(terms), _ptr(tot))
    return terms, float(tot[0])


def shuffle_keys(seed: int, rank: int, iteration: int, n_epochs: int, epoch: int):
    """SHUFFLE words 0..3 with id = rank, event = iteration*E + epoch."""
    ev = (iteration * n_epochs + epoch) & 0xFFFFFFFF
    return philox(seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF, [0, rank, ev, 6])


class Trainer:
    """The oracle's whole PPO iteration: T x (policy forward + Gaussian sample + env step,
    with the time-out bootstrap value of the pre-reset observation), GAE, E x K minibatch updates with
    Alg. 1 and Adam.  fp32 environment (C) + fp64 learning (numpy)."""

    def __init__(self, n_envs, n_steps, hf, n_levels, n_cols, theta, seed=0, scan=(17, 11), hidden=(512, 256, 128),
                 flags=F_CURRICULUM | F_NOISE | F_PUSH | F_BOOTSTRAP, n_epochs=5, n_minibatches=4, rank=0):
        self.env = Env(n_envs, hf, n_levels, n_cols, seed=seed, rank=rank, scan=scan, flags=flags)
        self.N, self.T, self.E, self.K = n_envs, n_steps, n_epochs, n_minibatches
        self.hidden, self.seed, self.rank, self.flags = hidden, seed, rank, flags
        self.D = self.env.obs_dim
        self.theta = np.asarray(theta, np.float64).copy()
        self.m = np.zeros_like(self.theta)
        self.v = np.zeros_like(self.theta)
        self.t_adam, self.alpha, self.iteration = 0, 1e-3, 0
        self.obs = self.env.reset()

    def _value(self, p, o):
        v, _ = learn.mlp_forward(p, np.asarray(o, np.float64), "c")
        return v[:, 0]

    def run_iteration(self):
        T, N, D = self.T, self.N, self.D
        p = learn.unpack(self.theta, D, self.hidden)
        ls = p["logstd"]
        bt = {k: np.zeros((T, N) + s, dt) for k, s, dt in
              (("obs", (D,), np.float32), ("act", (12,), np.float64), ("mu", (12,), np.float64), ("logp", (), np.float64),
               ("V", (), np.float64), ("r", (), np.float64), ("b", (), np.float64), ("term", (), np.uint8),
               ("timeout", (), np.uint8))}
        for t in range(T):
            o = self.obs
            mu, _ = learn.mlp_forward(p, o.astype(np.float64), "a")
            eps = self.env.action_eps()
            a = mu + np.exp(ls) * eps
            bt["obs"][t], bt["act"][t], bt["mu"][t] = o, a, mu
            bt["logp"][t] = learn.logp_gauss(a, mu, ls)
            bt["V"][t] = self._value(p, o)
            o2, r, te, to, _, tobs = self.env.step(a.astype(np.float32))
            bt["r"][t], bt["term"][t], bt["timeout"][t] = r, te, to
            if (self.flags & F_BOOTSTRAP) and to.any():
                bt["b"][t][to != 0] = self._value(p, tobs[to != 0])
            self.obs = o2
        bt["V_T"] = self._value(p, self.obs)
        bt["logstd_old"] = ls.copy()
        B = T * N
        perms = [feistel_perm(B, shuffle_keys(self.seed, self.rank, self.iteration, self.E, e)) for e in range(self.E)]
        self.theta, self.m, self.v, self.t_adam, self.alpha, stats = learn.ppo_update(
            self.theta, self.m, self.v, self.t_adam, self.alpha, bt, perms, D, self.hidden, n_epochs=self.E,
            n_minibatches=self.K, bootstrap=bool(self.flags & F_BOOTSTRAP))
        self.iteration += 1
        return stats
