"""ctypes binding of libleggedrl.so (include/lg.h) -- argument marshalling only.

Every function below has the name of the C entry point it wraps and forwards its arguments as plain
pointers/sizes; all computation happens in the CUDA library.  There is no fallback: importing this
module raises if the library has not been built (``python -m paper_2109_11978_b200.build``).
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# LG_LIB: another build of the same library (A/B timing of two builds in one process launch; diagnostics)
LIB_PATH = os.environ.get("LG_LIB") or os.path.join(HERE, "csrc", "libleggedrl.so")
NUM_BUFFERS = 20
BUF = dict(HEIGHTFIELD=0, STATE=1, OBS=2, ACT=3, MU=4, LOGP=5, VALUE=6, REWARD=7, BOOT=8, FLAGS=9, ADV=10, RET=11,
           VALUE_T=12, THETA=13, ADAM_M=14, ADAM_V=15, GRAD=16, WEIGHTS=17, ACTIV=18, WORK=19)
F_CURRICULUM, F_NOISE, F_PUSH, F_BOOTSTRAP, F_DETERMINISTIC = 1, 2, 4, 8, 32
F_UNFUSED_POLICY = 256  # diagnostics: per-layer rollout policy instead of the fused kernel (bit-identical)
F_UNFUSED_LOSS = 512  # diagnostics: layer-3 GEMM + separate loss-head kernel instead of the fused loss epilogue
STATUS = {0: "LG_OK", 1: "LG_ERR_INVALID_ARG", 2: "LG_ERR_RANGE", 3: "LG_ERR_SHAPE", 4: "LG_ERR_STATE",
          5: "LG_ERR_CUDA", 6: "LG_ERR_NCCL", 7: "LG_ERR_UNSUPPORTED"}


class lg_config(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("n_envs", ctypes.c_int32), ("n_steps", ctypes.c_int32),
                ("n_epochs", ctypes.c_int32), ("n_minibatches", ctypes.c_int32), ("hidden", ctypes.c_int32 * 3),
                ("scan_nx", ctypes.c_int32), ("scan_ny", ctypes.c_int32), ("n_levels", ctypes.c_int32),
                ("n_cols", ctypes.c_int32), ("inv_cell", ctypes.c_float), ("gamma", ctypes.c_float),
                ("lam", ctypes.c_float), ("clip", ctypes.c_float), ("vclip", ctypes.c_float),
                ("ent_coef", ctypes.c_float), ("vf_coef", ctypes.c_float), ("kl_target", ctypes.c_float),
                ("lr_init", ctypes.c_float), ("adam_b1", ctypes.c_float), ("adam_b2", ctypes.c_float),
                ("adam_eps", ctypes.c_float), ("seed", ctypes.c_uint64), ("rank", ctypes.c_int32),
                ("world_size", ctypes.c_int32), ("flags", ctypes.c_uint32)]


class lg_update_stats(ctypes.Structure):
    _fields_ = [("surrogate_loss", ctypes.c_float), ("value_loss", ctypes.c_float), ("entropy", ctypes.c_float),
                ("mean_kl", ctypes.c_float), ("lr", ctypes.c_float), ("clip_fraction", ctypes.c_float),
                ("nonfinite_skips", ctypes.c_int32), ("minibatches_applied", ctypes.c_int32),
                ("mean_episode_return", ctypes.c_float), ("mean_episode_length", ctypes.c_float),
                ("episodes", ctypes.c_int32), ("promotions", ctypes.c_int32), ("demotions", ctypes.c_int32),
                ("nonfinite_envs", ctypes.c_int32), ("level_hist", ctypes.c_int32 * 16)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "level_hist"}
        d["level_hist"] = list(self.level_hist)
        return d


EXPORTS = ["lg_num_params", "lg_obs_dim", "lg_obs_stride", "lg_required_sizes", "lg_create", "lg_destroy",
           "lg_last_error", "lg_params_set", "lg_params_sync", "lg_resume", "env_reset", "env_step_obs_reward", "policy_act",
           "policy_forward", "storage_compute_gae", "ppo_update", "ppo_shuffle", "ppo_minibatch_grad", "curriculum_update",
           "lg_nccl_unique_id", "lg_set_nccl", "lg_broadcast_params", "lg_iterate_host",
           "lg_graph_capture_iteration", "lg_graph_launch", "lg_device_scalars", "lg_profile", "lg_profile_read", "lg_graph_kernel_count",
           "lg_terrain_generate", "lg_group_create", "lg_group_destroy", "lg_group_broadcast_params",
           "lg_group_compute_gae", "lg_group_ppo_update", "lg_group_iterate", "lg_adv_normalization"]
MAX_GROUP = 8
PROF_CATS = ["env", "gemm_roll", "gemm_fwd", "gemm_dx", "gemm_dw", "heads", "loss", "reduce", "gather", "adam", "gae",
             "comm", "misc"]

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libleggedrl.so not built ({LIB_PATH}); run python -m paper_2109_11978_b200.build")
_lib = ctypes.CDLL(LIB_PATH)

P = ctypes.c_void_p
I32 = ctypes.c_int32
_sig = {
    "lg_num_params": (ctypes.c_int64, [ctypes.POINTER(lg_config)]),
    "lg_obs_dim": (I32, [ctypes.POINTER(lg_config)]),
    "lg_obs_stride": (I32, [ctypes.POINTER(lg_config)]),
    "lg_required_sizes": (I32, [ctypes.POINTER(lg_config), ctypes.POINTER(ctypes.c_size_t)]),
    "lg_create": (I32, [ctypes.POINTER(lg_config), ctypes.POINTER(P), P, ctypes.POINTER(P)]),
    "lg_destroy": (I32, [P]),
    "lg_last_error": (ctypes.c_char_p, [P]),
    "lg_params_set": (I32, [P, P]),
    "lg_params_sync": (I32, [P]),
    "lg_resume": (I32, [P]),
    "env_reset": (I32, [P, P, I32, P]),
    "env_step_obs_reward": (I32, [P, I32, P, P, P, P, P, P]),
    "policy_act": (I32, [P, I32, P, P, P, P]),
    "policy_forward": (I32, [P, P, I32, P, P]),
    "storage_compute_gae": (I32, [P, P, P]),
    "ppo_update": (I32, [P, P]),
    "ppo_minibatch_grad": (I32, [P, P, I32]),
    "ppo_shuffle": (I32, [P, I32, P]),
    "curriculum_update": (I32, [P, I32, P, P, P, P, P, P]),
    "lg_nccl_unique_id": (I32, [ctypes.c_char_p]),
    "lg_set_nccl": (I32, [P, ctypes.c_char_p]),
    "lg_broadcast_params": (I32, [P]),
    "lg_iterate_host": (I32, [P, ctypes.c_char_p, ctypes.POINTER(lg_update_stats)]),
    "lg_graph_capture_iteration": (I32, [P, P]),
    "lg_graph_launch": (I32, [P]),
    "lg_device_scalars": (I32, [P, ctypes.POINTER(I32)]),
    "lg_profile": (I32, [P, I32]),
    "lg_graph_kernel_count": (I32, [P, ctypes.POINTER(I32)]),
    "lg_profile_read": (I32, [P, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(I32), I32]),
    "lg_terrain_generate": (I32, [P, I32, I32, ctypes.c_uint64, P]),
    "lg_adv_normalization": (I32, [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    "lg_group_create": (I32, [ctypes.POINTER(P), I32, ctypes.POINTER(P)]),
    "lg_group_destroy": (I32, [P]),
    "lg_group_broadcast_params": (I32, [P]),
    "lg_group_compute_gae": (I32, [P]),
    "lg_group_ppo_update": (I32, [P, ctypes.POINTER(P)]),
    "lg_group_iterate": (I32, [P, ctypes.POINTER(P)]),
}
for _n, (_r, _a) in _sig.items():
    _f = getattr(_lib, _n)
    _f.restype = _r
    _f.argtypes = _a


class LgError(RuntimeError):
    pass


def check(status, ctx=None, what=""):
    if status != 0:
        msg = _lib.lg_last_error(ctx).decode() if ctx else ""
        raise LgError(f"{what}: {STATUS.get(status, status)} {msg}")


def _p(x):
    """device pointer of a torch tensor (or None/int passthrough)"""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


# ---- thin wrappers with the C names ------------------------------------------------------------
def lg_num_params(cfg):
    return _lib.lg_num_params(ctypes.byref(cfg))


def lg_obs_dim(cfg):
    return _lib.lg_obs_dim(ctypes.byref(cfg))


def lg_obs_stride(cfg):
    return _lib.lg_obs_stride(ctypes.byref(cfg))


def lg_terrain_generate(hf, n_levels, n_cols, seed, stream=None):
    """World heightfield into the fp32 device tensor hf [80 L][80 C] (include/lg.h)."""
    if tuple(hf.shape) != (80 * n_levels, 80 * n_cols) or not hf.is_contiguous() or str(hf.dtype) != "torch.float32":
        raise LgError("lg_terrain_generate: hf must be a contiguous fp32 [80 L][80 C] device tensor")
    check(_lib.lg_terrain_generate(_p(hf), n_levels, n_cols, seed & 0xFFFFFFFFFFFFFFFF, stream), None,
          "lg_terrain_generate")


def lg_required_sizes(cfg):
    arr = (ctypes.c_size_t * NUM_BUFFERS)()
    st = _lib.lg_required_sizes(ctypes.byref(cfg), arr)
    return st, list(arr)


def lg_create(cfg, buffers, stream_handle):
    arr = (P * NUM_BUFFERS)(*[_p(b) for b in buffers])
    out = P()
    st = _lib.lg_create(ctypes.byref(cfg), arr, P(stream_handle), ctypes.byref(out))
    return st, out


def lg_destroy(ctx):
    return _lib.lg_destroy(ctx)


def lg_last_error(ctx):
    return _lib.lg_last_error(ctx).decode()


def lg_params_set(ctx, theta):
    return _lib.lg_params_set(ctx, _p(theta))


def lg_params_sync(ctx):
    return _lib.lg_params_sync(ctx)


def lg_resume(ctx):
    return _lib.lg_resume(ctx)


def env_reset(ctx, mask=None, init=1, obs=None):
    return _lib.env_reset(ctx, _p(mask), int(init), _p(obs))


def env_step_obs_reward(ctx, t, actions=None, obs=None, reward=None, terminated=None, timeout=None, terms=None):
    return _lib.env_step_obs_reward(ctx, int(t), _p(actions), _p(obs), _p(reward), _p(terminated), _p(timeout),
                                    _p(terms))


def policy_act(ctx, t, actions=None, logp=None, mu=None, value=None):
    return _lib.policy_act(ctx, int(t), _p(actions), _p(logp), _p(mu), _p(value))


def policy_forward(ctx, x, M, mu, value):
    return _lib.policy_forward(ctx, _p(x), int(M), _p(mu), _p(value))


def storage_compute_gae(ctx, adv=None, ret=None):
    return _lib.storage_compute_gae(ctx, _p(adv), _p(ret))


def ppo_update(ctx, stats=None):
    return _lib.ppo_update(ctx, _p(stats))


def ppo_shuffle(ctx, epoch, perm):
    return _lib.ppo_shuffle(ctx, int(epoch), _p(perm))


def ppo_minibatch_grad(ctx, idx, M_mb):
    return _lib.ppo_minibatch_grad(ctx, _p(idx), int(M_mb))


def curriculum_update(ctx, n, crossed, disp_xy, cmd_xy, ep_steps, loop_words, level):
    return _lib.curriculum_update(ctx, int(n), _p(crossed), _p(disp_xy), _p(cmd_xy), _p(ep_steps), _p(loop_words),
                                  _p(level))


def lg_nccl_unique_id():
    buf = ctypes.create_string_buffer(128)
    st = _lib.lg_nccl_unique_id(buf)
    return st, bytes(buf.raw)


def lg_set_nccl(ctx, uid: bytes):
    return _lib.lg_set_nccl(ctx, uid)


def lg_broadcast_params(ctx):
    return _lib.lg_broadcast_params(ctx)


def lg_iterate_host(ctx, ctrl: bytes, stats: lg_update_stats):
    return _lib.lg_iterate_host(ctx, ctrl, ctypes.byref(stats))


def lg_graph_capture_iteration(ctx, stats=None):
    return _lib.lg_graph_capture_iteration(ctx, _p(stats))


def lg_graph_launch(ctx):
    return _lib.lg_graph_launch(ctx)


def lg_device_scalars(ctx):
    out = (I32 * 8)()
    st = _lib.lg_device_scalars(ctx, out)
    return st, list(out)


def lg_profile(ctx, enable):
    return _lib.lg_profile(ctx, int(enable))


def lg_profile_read(ctx):
    n = len(PROF_CATS)
    ms = (ctypes.c_float * n)()
    cnt = (I32 * n)()
    st = _lib.lg_profile_read(ctx, ms, cnt, n)
    return st, list(ms), list(cnt)


def lg_graph_kernel_count(ctx):
    n = I32()
    st = _lib.lg_graph_kernel_count(ctx, ctypes.byref(n))
    return st, n.value


def lg_group_create(ctxs):
    arr = (P * len(ctxs))(*[c.value if isinstance(c, P) else c for c in ctxs])
    out = P()
    st = _lib.lg_group_create(arr, len(ctxs), ctypes.byref(out))
    return st, out


def lg_group_destroy(g):
    return _lib.lg_group_destroy(g)


def lg_group_broadcast_params(g):
    return _lib.lg_group_broadcast_params(g)


def lg_group_compute_gae(g):
    return _lib.lg_group_compute_gae(g)


def _stats_arr(stats):
    if stats is None:
        return None
    return (P * len(stats))(*[_p(s) for s in stats])


def lg_group_ppo_update(g, stats=None):
    return _lib.lg_group_ppo_update(g, _stats_arr(stats))


def lg_group_iterate(g, stats=None):
    return _lib.lg_group_iterate(g, _stats_arr(stats))


def lg_adv_normalization(ctx):
    m, i = ctypes.c_double(), ctypes.c_double()
    st = _lib.lg_adv_normalization(ctx, ctypes.byref(m), ctypes.byref(i))
    return st, m.value, i.value
