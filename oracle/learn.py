"""oracle/learn.py -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Plain fp64 numpy implementation of the learning side of the hot path: actor-critic MLP forward and
exact reverse-mode backward, diagonal-Gaussian log-probabilities, GAE with time-out bootstrapping,
advantage normalisation, the clipped-surrogate PPO loss with clipped value loss and entropy bonus,
the analytic KL, Algorithm 1 (adaptive learning rate) and Adam.  Written from DESIGN.md §3.8-§3.11,
which restate PAPER.md §2.2, Table 3, Alg. 1 and SPEC.md's net/ppo
modules.  numpy matmul is the only library primitive used as a step.

Pins (tests/test_oracle_learn.py): GAE vs brute-force truncated sums and S:421-422 examples and the
closed forms of SURVEY §8(c).3; PPO loss at ratio = 1 vs closed form; Alg. 1 examples
(S:439-442); Adam first-step closed form; logp/entropy constants; MLP backward vs
central finite differences; zero-weight net outputs zero.
"""
from __future__ import annotations

import math

import numpy as np

LOG_2PI = math.log(2.0 * math.pi)


# ----------------------------------------------------------------------------------------------
# Parameter layout: actor W1,b1,W2,b2,W3,b3,W4,b4; critic (same); log-std.
# ----------------------------------------------------------------------------------------------
def param_shapes(obs_dim: int, hidden=(512, 256, 128), act_dim: int = 12):
    shapes = []
    for net, out in (("a", act_dim), ("c", 1)):
        dims = [obs_dim, *hidden, out]
        for l in range(4):
            shapes.append((f"{net}W{l + 1}", (dims[l + 1], dims[l])))
            shapes.append((f"{net}b{l + 1}", (dims[l + 1],)))
    shapes.append(("logstd", (act_dim,)))
    return shapes


def num_params(obs_dim: int, hidden=(512, 256, 128), act_dim: int = 12) -> int:
    return int(sum(np.prod(s) for _, s in param_shapes(obs_dim, hidden, act_dim)))


def unpack(theta: np.ndarray, obs_dim: int, hidden=(512, 256, 128), act_dim: int = 12) -> dict:
    out, o = {}, 0
    for name, shp in param_shapes(obs_dim, hidden, act_dim):
        n = int(np.prod(shp))
        out[name] = np.asarray(theta[o:o + n], dtype=np.float64).reshape(shp)
        o += n
    assert o == theta.size
    return out


def pack(p: dict, obs_dim: int, hidden=(512, 256, 128), act_dim: int = 12) -> np.ndarray:
    return np.concatenate([p[name].reshape(-1) for name, _ in param_shapes(obs_dim, hidden, act_dim)])


# ----------------------------------------------------------------------------------------------
# MLP (BJ 512-256-128 ELU)
# ----------------------------------------------------------------------------------------------
def round_bf16(x):
    """Round-to-nearest-even to bfloat16 of the fp32 rounding of x (R26 / SURVEY §8(c).1's
    diagnostic switch: the GEMM operand rounding points of the GPU path), returned as fp64."""
    b = np.ascontiguousarray(np.asarray(x, np.float64).astype(np.float32)).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32).astype(np.float64).reshape(np.shape(x))


def round_tf32(x):
    """Round-to-nearest-even to TF32 (10 explicit mantissa bits) of the fp32 rounding of x, as fp64."""
    b = np.ascontiguousarray(np.asarray(x, np.float64).astype(np.float32)).view(np.uint32).astype(np.uint64)
    b = (b + 0xFFF + ((b >> 13) & 1)) & 0xFFFFE000
    return b.astype(np.uint32).view(np.float32).astype(np.float64).reshape(np.shape(x))


def round_fp32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


_ROUND = {"bf16": round_bf16, "tf32": round_tf32, "fp32": round_fp32}


def _q(x, quant, point=None):
    """Rounding of a GEMM operand at one of the GPU path's rounding points (SURVEY §8(c).1 diagnostic switch).
    quant: None (exact fp64), "bf16" / "tf32" / "fp32" (every point), or "<format>@<point>" (that point only);
    points: "w" forward weights, "h" stored activations (incl. the input rows), "dz" stored pre-activation
    gradients, "wb" weights of the input-gradient products."""
    if quant is None:
        return x
    fmt, _, only = quant.partition("@")
    if only and point != only:
        return x
    return _ROUND[fmt](x)


def elu(x):
    return np.where(x > 0, x, np.expm1(np.minimum(x, 0.0)))


def mlp_forward(p: dict, x: np.ndarray, net: str, quant=None):
    """Returns output and the list of layer inputs/outputs needed by the backward pass.
    quant='bf16' rounds the hidden-layer weights and the stored activations to bf16 (GPU rounding points)."""
    x = _q(x, quant, "h")
    acts = [x]
    h = x
    for l in range(1, 4):
        h = _q(elu(h @ _q(p[f"{net}W{l}"], quant, "w").T + p[f"{net}b{l}"]), quant, "h")
        acts.append(h)
    y = h @ p[f"{net}W4"].T + p[f"{net}b4"]
    return y, acts


def mlp_backward(p: dict, acts, dy: np.ndarray, net: str, grads: dict, quant=None):
    """Exact reverse mode for y = W4 ELU(W3 ELU(W2 ELU(W1 x + b1) + b2) + b3) + b4.
    ELU'(z) = 1 if out > 0 else out + 1 (= exp z), so only layer outputs are needed.
    quant='bf16' also rounds each dZ_l = dH_l * ELU'(H_l) and the hidden weights used for dX to bf16."""
    g = dy
    for l in range(4, 0, -1):
        a_in = acts[l - 1]
        grads[f"{net}W{l}"] = g.T @ a_in
        grads[f"{net}b{l}"] = g.sum(axis=0)
        if l > 1:
            g = g @ (p[f"{net}W{l}"] if l == 4 else _q(p[f"{net}W{l}"], quant, "wb"))
            out = acts[l - 1]
            g = _q(g * np.where(out > 0, 1.0, out + 1.0), quant, "dz")


def logp_gauss(a, mu, logstd):
    """logp(a|mu,sigma) = -sum_j [0.5((a_j-mu_j)e^{-l_j})^2 + l_j] - (A/2) ln 2pi."""
    z = (a - mu) * np.exp(-logstd)
    return -(0.5 * z * z + logstd).sum(axis=-1) - 0.5 * a.shape[-1] * LOG_2PI


def entropy_gauss(logstd):
    return float(np.sum(0.5 + 0.5 * LOG_2PI + logstd))


# ----------------------------------------------------------------------------------------------
# GAE with time-out bootstrapping
# ----------------------------------------------------------------------------------------------
def gae(r, V, V_T, b, term, timeout, gamma=0.99, lam=0.95, bootstrap=True):
    """r, V, b, term, timeout: [T][N]; V_T: [N]. Returns (A, R) fp64 [T][N]."""
    r = np.asarray(r, np.float64)
    V = np.asarray(V, np.float64)
    T, N = r.shape
    A = np.zeros((T, N))
    nextA = np.zeros(N)
    nextV = np.asarray(V_T, np.float64)
    for t in range(T - 1, -1, -1):
        done = (np.asarray(term[t]) != 0) | (np.asarray(timeout[t]) != 0)
        nd = 1.0 - done.astype(np.float64)
        rt = r[t] + (gamma * np.asarray(b[t], np.float64) if bootstrap else 0.0)
        delta = rt + gamma * nd * nextV - V[t]
        A[t] = delta + gamma * lam * nd * nextA
        nextA = A[t]
        nextV = V[t]
    return A, A + V


def normalize_adv(A):
    A = np.asarray(A, np.float64)
    return (A - A.mean()) / (A.std(ddof=1) + 1e-8)


# ----------------------------------------------------------------------------------------------
# PPO loss + gradients on one minibatch (Table 3)
# ----------------------------------------------------------------------------------------------
def ppo_minibatch(p: dict, obs, act, logp_old, V_old, adv_n, ret, mu_old, logstd_old,
                  clip=0.2, vclip=0.2, ent_coef=0.01, vf_coef=1.0, quant=None):
    """Returns (grads dict, stats dict). adv_n = normalised advantages."""
    M = obs.shape[0]
    mu, acts_a = mlp_forward(p, obs, "a", quant)
    v, acts_c = mlp_forward(p, obs, "c", quant)
    v = v[:, 0]
    ls = p["logstd"]
    sig2 = np.exp(2.0 * ls)
    logp = logp_gauss(act, mu, ls)
    rho = np.exp(logp - logp_old)
    s1 = rho * adv_n
    rc = np.clip(rho, 1.0 - clip, 1.0 + clip)
    s2 = rc * adv_n
    take1 = s1 <= s2
    L_pi = -np.mean(np.where(take1, s1, s2))
    vc = V_old + np.clip(v - V_old, -vclip, vclip)
    e1 = (v - ret) ** 2
    e2 = (vc - ret) ** 2
    take_u = e1 >= e2
    L_V = np.mean(np.where(take_u, e1, e2))
    H = entropy_gauss(ls)
    loss = L_pi + vf_coef * L_V - ent_coef * H
    sig2_old = np.exp(2.0 * logstd_old)
    kl = np.mean(np.sum(ls - logstd_old + (sig2_old + (mu_old - mu) ** 2) / (2.0 * sig2) - 0.5, axis=1))
    # d loss / d rho
    inside = (rho >= 1.0 - clip) & (rho <= 1.0 + clip)
    dL_drho = -np.where(take1, adv_n, adv_n * inside) / M
    dL_dlogp = dL_drho * rho
    diff = act - mu
    dmu = dL_dlogp[:, None] * diff / sig2
    dls = np.sum(dL_dlogp[:, None] * (diff * diff / sig2 - 1.0), axis=0) - ent_coef
    vin = np.abs(v - V_old) <= vclip
    dV = vf_coef * np.where(take_u, 2.0 * (v - ret), 2.0 * (vc - ret) * vin) / M
    grads = {}
    mlp_backward(p, acts_a, dmu, "a", grads, quant)
    mlp_backward(p, acts_c, dV[:, None], "c", grads, quant)
    grads["logstd"] = dls
    stats = dict(loss=loss, surrogate=L_pi, value_loss=L_V, entropy=H, kl=kl,
                 clip_frac=float(np.mean(np.abs(rho - 1.0) > clip)))
    return grads, stats


def alg1(kl: float, alpha: float, kl_target: float = 0.01) -> float:
    """Algorithm 1."""
    if kl > 2.0 * kl_target:
        return max(1e-5, alpha / 1.5)
    if kl < 0.5 * kl_target:
        return min(1e-2, 1.5 * alpha)
    return alpha


def adam_step(theta, g, m, v, t, alpha, b1=0.9, b2=0.999, eps=1e-8):
    """One bias-corrected Adam step. Returns (theta, m, v, t)."""
    t = t + 1
    m = b1 * m + (1.0 - b1) * g
    v = b2 * v + (1.0 - b2) * g * g
    mh = m / (1.0 - b1 ** t)
    vh = v / (1.0 - b2 ** t)
    theta = theta - alpha * mh / (np.sqrt(vh) + eps)
    return theta, m, v, t


def ppo_update(theta, m, v, t_adam, alpha, batch: dict, perms, obs_dim, hidden=(512, 256, 128),
               n_epochs=5, n_minibatches=4, gamma=0.99, lam=0.95, bootstrap=True, kl_target=0.01, quant=None):
    """One PPO update on a collected batch.

    batch: obs [T][N][D], act/mu [T][N][12], logp, V, r, b [T][N], term/timeout [T][N], V_T [N],
    logstd_old [12].  perms: list over epochs of permutations of [0, T*N).
    Returns (theta, m, v, t_adam, alpha, stats list)."""
    T, N = batch["r"].shape
    B = T * N
    A, Ret = gae(batch["r"], batch["V"], batch["V_T"], batch["b"], batch["term"], batch["timeout"],
                 gamma, lam, bootstrap)
    An = normalize_adv(A).reshape(B)
    Ret = Ret.reshape(B)
    obs = np.asarray(batch["obs"], np.float64).reshape(B, -1)[:, :obs_dim]
    act = np.asarray(batch["act"], np.float64).reshape(B, -1)
    mu_old = np.asarray(batch["mu"], np.float64).reshape(B, -1)
    logp_old = np.asarray(batch["logp"], np.float64).reshape(B)
    V_old = np.asarray(batch["V"], np.float64).reshape(B)
    ls_old = np.asarray(batch["logstd_old"], np.float64)
    Mb = B // n_minibatches
    theta = np.asarray(theta, np.float64).copy()
    stats = []
    for e in range(n_epochs):
        pe = np.asarray(perms[e], np.int64)
        for k in range(n_minibatches):
            idx = pe[k * Mb:(k + 1) * Mb]
            p = unpack(theta, obs_dim, hidden)
            g, st = ppo_minibatch(p, obs[idx], act[idx], logp_old[idx], V_old[idx], An[idx], Ret[idx],
                                  mu_old[idx], ls_old, quant=quant)
            gflat = pack(g, obs_dim, hidden)
            if not (np.isfinite(st["loss"]) and np.all(np.isfinite(gflat))):
                st["skipped"] = True
                stats.append(st)
                continue
            alpha = alg1(st["kl"], alpha, kl_target)
            theta, m, v, t_adam = adam_step(theta, gflat, m, v, t_adam, alpha)
            st["alpha"] = alpha
            stats.append(st)
    return theta, m, v, t_adam, alpha, stats


def ppo_update_union(theta, m, v, t_adam, alpha, batches: list, perms: list, obs_dim, hidden=(512, 256, 128),
                     n_epochs=5, n_minibatches=4, gamma=0.99, lam=0.95, bootstrap=True, kl_target=0.01, quant=None):
    """One PPO update over W ranks' batches with the multi-rank semantics of SURVEY §8(c).1 O-M:
    GAE per rank; advantages normalised over the union of all ranks' samples (R13); the global minibatch (e, k)
    is the union, in rank order, of every rank's minibatch k of epoch e under that rank's own permutation
    perms[r][e]; the gradient is that of the union minibatch's mean loss and the KL its mean (so Alg. 1 and
    Adam act identically on every replica).  batches[r] / perms[r] as in ppo_update.  With W = 1 this is
    ppo_update.  Returns (theta, m, v, t_adam, alpha, stats list)."""
    W = len(batches)
    T, N = batches[0]["r"].shape
    B = T * N
    cols = {k: [] for k in ("obs", "act", "mu", "logp", "V", "A", "R")}
    for bt in batches:
        A, Ret = gae(bt["r"], bt["V"], bt["V_T"], bt["b"], bt["term"], bt["timeout"], gamma, lam, bootstrap)
        cols["A"].append(A.reshape(B))
        cols["R"].append(Ret.reshape(B))
        cols["obs"].append(np.asarray(bt["obs"], np.float64).reshape(B, -1)[:, :obs_dim])
        cols["act"].append(np.asarray(bt["act"], np.float64).reshape(B, -1))
        cols["mu"].append(np.asarray(bt["mu"], np.float64).reshape(B, -1))
        cols["logp"].append(np.asarray(bt["logp"], np.float64).reshape(B))
        cols["V"].append(np.asarray(bt["V"], np.float64).reshape(B))
    An = normalize_adv(np.concatenate(cols["A"])).reshape(W, B)  # union statistics
    ls_old = np.asarray(batches[0]["logstd_old"], np.float64)
    Mb = B // n_minibatches
    theta = np.asarray(theta, np.float64).copy()
    stats = []
    for e in range(n_epochs):
        for k in range(n_minibatches):
            idx = [np.asarray(perms[r][e], np.int64)[k * Mb:(k + 1) * Mb] for r in range(W)]
            u = lambda name: np.concatenate([cols[name][r][idx[r]] for r in range(W)])  # noqa: E731
            adv = np.concatenate([An[r][idx[r]] for r in range(W)])
            p = unpack(theta, obs_dim, hidden)
            g, st = ppo_minibatch(p, u("obs"), u("act"), u("logp"), u("V"), adv, u("R"), u("mu"), ls_old, quant=quant)
            gflat = pack(g, obs_dim, hidden)
            if not (np.isfinite(st["loss"]) and np.all(np.isfinite(gflat))):
                st["skipped"] = True
                stats.append(st)
                continue
            alpha = alg1(st["kl"], alpha, kl_target)
            theta, m, v, t_adam = adam_step(theta, gflat, m, v, t_adam, alpha)
            st["alpha"] = alpha
            stats.append(st)
    return theta, m, v, t_adam, alpha, stats
