"""Pins for the learning side of the oracle (oracle/learn.py) against the paper's worked examples,
closed forms, brute force and finite differences.  CPU only."""
import math
import os

import numpy as np
import pytest

from oracle import learn
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


# ---------------------------------------------------------------- Alg. 1
def test_alg1_examples_bit_exact():
    for kl, a_in, a_out in _rows("alg1_examples.txt"):
        got = learn.alg1(float(kl), float(a_in))
        assert abs(got - float(a_out)) <= 1e-15 * float(a_out)     # printed decimal, within 1 ulp
        assert got in (float(a_in) / 1.5, max(1e-5, float(a_in) / 1.5), 1.5 * float(a_in), float(a_in))


def test_alg1_bounds_fuzz():
    rng = np.random.default_rng(0)
    a = 1e-3
    for _ in range(10000):
        a = learn.alg1(float(rng.exponential(0.01)), a)
        assert 1e-5 <= a <= 1e-2
    assert learn.alg1(0.0, 1e-3) == 1.5e-3                     # first minibatch of an iteration: KL = 0


# ---------------------------------------------------------------- GAE
def test_gae_spec_examples():
    for r, V, b, term, to, A_exp in _rows("gae_examples.txt"):
        A, R = learn.gae([[float(r)]], [[float(V)]], [0.0], [[float(b)]], [[int(term)]], [[int(to)]])
        assert abs(A[0, 0] - float(A_exp)) < 1e-12
        assert abs(R[0, 0] - (float(A_exp) + float(V))) < 1e-12


def test_gae_worked_vector_and_bootstrap_off():
    # SURVEY §8(c).5 (hand-derived): γ=0.99, λ=0.95, T=4
    r = np.array([[1.0], [0.5], [-0.2], [2.0]])
    V = np.array([[0.3], [0.6], [0.1], [0.4]])
    term = np.array([[0], [0], [1], [0]])
    to = np.array([[1], [0], [0], [0]])
    b = np.array([[2.0], [0], [0], [0]])
    A, R = learn.gae(r, V, [0.7], b, term, to)
    assert np.allclose(A[:, 0], [2.68, -0.28315, -0.3, 2.293], atol=1e-12)
    assert np.allclose(R[:, 0], [2.98, 0.31685, -0.2, 2.693], atol=1e-12)
    A0, _ = learn.gae(r, V, [0.7], b, term, to, bootstrap=False)
    assert abs(A0[0, 0] - 0.7) < 1e-12
    An = learn.normalize_adv(A[:, 0])
    assert np.allclose(An, [0.98190597, -0.85661897, -0.86707378, 0.74178678], atol=1e-7)


def _brute_gae(r, V, VT, b, term, to, g, lam, boot=True):
    """A_t = Σ_{k=t}^{e} (γλ)^{k-t} δ_k, e = first k >= t with done_k (else T-1) -- S:423."""
    T, N = r.shape
    A = np.zeros((T, N))
    for i in range(N):
        for t in range(T):
            acc = 0.0
            for k in range(t, T):
                done = term[k, i] or to[k, i]
                vnext = 0.0 if done else (V[k + 1, i] if k + 1 < T else VT[i])
                rt = r[k, i] + (g * b[k, i] if boot else 0.0)
                acc += (g * lam) ** (k - t) * (rt + g * vnext - V[k, i])
                if done:
                    break
            A[t, i] = acc
    return A


def test_gae_brute_force_random_buffers():
    rng = np.random.default_rng(0)
    for trial in range(1000):
        T, N = int(rng.integers(1, 17)), int(rng.integers(1, 5))
        r, V = rng.standard_normal((T, N)), rng.standard_normal((T, N))
        VT, b = rng.standard_normal(N), rng.standard_normal((T, N))
        term = (rng.random((T, N)) < 0.2).astype(int)
        to = ((rng.random((T, N)) < 0.2) & (term == 0)).astype(int)
        boot = bool(trial % 2)
        A, _ = learn.gae(r, V, VT, b, term, to, 0.99, 0.95, boot)
        assert np.max(np.abs(A - _brute_gae(r, V, VT, b, term, to, 0.99, 0.95, boot))) < 1e-9


def test_gae_closed_forms():
    rng = np.random.default_rng(1)
    T, N = 12, 3
    r, V, VT = rng.standard_normal((T, N)), rng.standard_normal((T, N)), rng.standard_normal(N)
    z = np.zeros((T, N), int)
    A, _ = learn.gae(r, V, VT, np.zeros((T, N)), z, z, 0.99, 0.0)          # λ = 0 -> A = δ
    Vn = np.vstack([V[1:], VT[None]])
    assert np.allclose(A, r + 0.99 * Vn - V, atol=1e-12)
    A, _ = learn.gae(r, np.zeros((T, N)), np.zeros(N), np.zeros((T, N)), z, z, 1.0, 1.0)
    assert np.allclose(A, np.cumsum(r[::-1], axis=0)[::-1], atol=1e-12)   # reverse cumulative sum
    # constant δ, no dones: A_t = δ (1 - (γλ)^{T-t}) / (1 - γλ)
    d, g, lam = 0.3, 0.99, 0.95
    A, _ = learn.gae(np.full((T, 1), d), np.zeros((T, 1)), np.zeros(1), np.zeros((T, 1)), z[:, :1], z[:, :1], g, lam)
    gl = g * lam
    assert np.allclose(A[:, 0], [d * (1 - gl ** (T - t)) / (1 - gl) for t in range(T)], atol=1e-12)
    # bootstrap off == time-outs treated as terminations
    to = (rng.random((T, N)) < 0.3).astype(int)
    b = rng.standard_normal((T, N))
    A1, _ = learn.gae(r, V, VT, b, z, to, bootstrap=False)
    A2, _ = learn.gae(r, V, VT, np.zeros((T, N)), to, z, bootstrap=True)
    assert np.allclose(A1, A2, atol=1e-12)


def test_normalized_advantages_moments():
    a = learn.normalize_adv(np.random.default_rng(2).standard_normal(1000) * 3 + 5)
    assert abs(a.mean()) < 1e-12 and abs(a.std(ddof=1) - 1) < 1e-8


# ---------------------------------------------------------------- Gaussian policy
def test_logp_entropy_constants():
    assert abs(learn.logp_gauss(np.zeros(12), np.zeros(12), np.zeros(12)) - (-6 * math.log(2 * math.pi))) < 1e-12
    assert abs(learn.logp_gauss(np.zeros(12), np.zeros(12), np.zeros(12)) + 11.027262398) < 1e-8
    assert abs(learn.entropy_gauss(np.zeros(12)) - 17.027262398) < 1e-8
    # log-std -> -10 ~ deterministic
    mu = np.arange(12.0)
    lp_at_mu = learn.logp_gauss(mu, mu, np.full(12, -10.0))
    assert abs(lp_at_mu - (120.0 - 6 * math.log(2 * math.pi))) < 1e-9


# ---------------------------------------------------------------- MLP
def test_param_counts():
    assert learn.num_params(235) == 571801
    assert learn.num_params(48) == 380313
    assert learn.num_params(48, (128, 64, 32)) == 33657


def test_zero_net_outputs_zero_and_hand_unit():
    p = learn.unpack(np.zeros(learn.num_params(5, (1, 1, 1))), 5, (1, 1, 1))
    y, _ = learn.mlp_forward(p, np.random.default_rng(0).standard_normal((3, 5)), "a")
    assert np.all(y == 0)
    # single hidden unit chain with hand weights: x=(1,2,0,0,0), W1 row (0.5,-1,...), b1=0.25 -> z=-1.25
    p["aW1"][0, :2] = [0.5, -1.0]
    p["ab1"][0] = 0.25
    p["aW2"][0, 0] = 2.0
    p["aW3"][0, 0] = 1.0
    p["aW4"][:, 0] = 3.0
    p["ab4"][:] = 0.1
    y, _ = learn.mlp_forward(p, np.array([[1.0, 2.0, 0, 0, 0]]), "a")
    h1 = math.expm1(-1.25)
    h2 = math.expm1(2 * h1)
    h3 = math.expm1(h2)
    assert np.allclose(y, 3 * h3 + 0.1, atol=1e-14)


def _tiny_batch(rng, M, D):
    return dict(obs=rng.standard_normal((M, D)), act=rng.standard_normal((M, 12)),
                logp_old=-17 + rng.standard_normal(M), V_old=rng.standard_normal(M),
                adv_n=rng.standard_normal(M), ret=rng.standard_normal(M),
                mu_old=0.3 * rng.standard_normal((M, 12)), logstd_old=0.1 * rng.standard_normal(12))


def test_backward_matches_finite_differences():
    """analytic gradient of the full PPO loss vs central differences (fp64)."""
    rng = np.random.default_rng(3)
    D, hid = 6, (5, 4, 3)
    theta = synth.init_params(D, hid, seed=4).astype(np.float64)
    theta[-12:] = 0.2 * rng.standard_normal(12)
    bt = _tiny_batch(rng, 9, D)
    bt["logp_old"] = learn.logp_gauss(bt["act"], bt["mu_old"], bt["logstd_old"]) + 0.05 * rng.standard_normal(9)

    def loss(th):
        _, st = learn.ppo_minibatch(learn.unpack(th, D, hid), **bt)
        return st["loss"]

    g, _ = learn.ppo_minibatch(learn.unpack(theta, D, hid), **bt)
    gflat = learn.pack(g, D, hid)
    h = 1e-6
    idx = rng.choice(theta.size, 80, replace=False)
    for k in idx:
        e = np.zeros_like(theta)
        e[k] = h
        fd = (loss(theta + e) - loss(theta - e)) / (2 * h)
        assert abs(fd - gflat[k]) <= 1e-6 * max(1.0, abs(fd))


def test_ppo_loss_at_ratio_one_closed_form():
    """θ = θ_old -> ρ = 1, KL = 0, L_π = −mean(Â), ∂L_π/∂μ = −Â(a−μ)/σ²/M."""
    rng = np.random.default_rng(5)
    D, hid, M = 7, (6, 5, 4), 50
    theta = synth.init_params(D, hid, seed=6).astype(np.float64)
    p = learn.unpack(theta, D, hid)
    obs = rng.standard_normal((M, D))
    mu, _ = learn.mlp_forward(p, obs, "a")
    v, _ = learn.mlp_forward(p, obs, "c")
    act = mu + rng.standard_normal((M, 12))
    adv = rng.standard_normal(M)
    ret = v[:, 0] + rng.standard_normal(M)
    g, st = learn.ppo_minibatch(p, obs, act, learn.logp_gauss(act, mu, p["logstd"]), v[:, 0], adv, ret, mu,
                                p["logstd"])
    assert abs(st["surrogate"] + adv.mean()) < 1e-12
    assert abs(st["kl"]) < 1e-12 and st["clip_frac"] == 0.0
    assert abs(st["value_loss"] - np.mean((v[:, 0] - ret) ** 2)) < 1e-12       # = MSE at V = V_old
    dmu = -adv[:, None] * (act - mu) / M                                        # σ = 1
    assert np.allclose(g["ab4"], dmu.sum(0), atol=1e-12)
    # clipping zeroes the gradient for Â > 0, ρ > 1.2
    lp_old = learn.logp_gauss(act, mu, p["logstd"]) - 1.0                      # ρ = e > 1.2
    g2, _ = learn.ppo_minibatch(p, obs, act, lp_old, v[:, 0], np.abs(adv), ret, mu, p["logstd"])
    assert np.allclose(g2["ab4"], 0.0, atol=1e-15)


def test_kl_analytic_example():
    """Δμ = 0.1 in all 12 dims, σ_old = σ = 1 -> KL = 0.06."""
    D, hid = 3, (2, 2, 2)
    p = learn.unpack(np.zeros(learn.num_params(D, hid)), D, hid)
    obs = np.zeros((4, D))
    _, st = learn.ppo_minibatch(p, obs, np.zeros((4, 12)), np.zeros(4), np.zeros(4), np.zeros(4), np.zeros(4),
                                np.full((4, 12), 0.1), np.zeros(12))
    assert abs(st["kl"] - 0.06) < 1e-12


# ---------------------------------------------------------------- Adam
def test_adam_closed_forms():
    th = np.array([1.0, -2.0, 3.0])
    z = np.zeros(3)
    t1, *_ = learn.adam_step(th, z, z, z, 0, 1e-3)
    assert np.array_equal(t1, th)                                # zero gradient
    g = np.array([0.5, -0.25, 1e-3])
    t1, m, v, t = learn.adam_step(th, g, z, z, 0, 1e-3)
    assert np.allclose(t1 - th, -1e-3 * g / (np.abs(g) + 1e-8), atol=1e-15)  # first step
    assert abs((t1 - th)[0] + 0.00099999998) < 1e-12
    t1, *_ = learn.adam_step(th, g, z, z, 0, 0.0)
    assert np.array_equal(t1, th)                                # α = 0


def test_ppo_update_runs_and_reduces_value_loss():
    """one full update on a fixed synthetic buffer reduces value loss."""
    import oracle
    D, hid = 10, (16, 16, 8)
    T, N = 8, 16
    bt = synth.synthetic_storage(T, N, D, seed=1)
    theta = synth.init_params(D, hid, seed=2).astype(np.float64)
    perms = [oracle.feistel_perm(T * N, oracle.shuffle_keys(0, 0, 0, 5, e)) for e in range(5)]
    m = np.zeros_like(theta)
    v = np.zeros_like(theta)
    th2, m, v, t, alpha, stats = learn.ppo_update(theta, m, v, 0, 1e-3, bt, perms, D, hid)
    assert t == 20 and len(stats) == 20
    assert stats[-1]["value_loss"] < stats[0]["value_loss"]
    assert 1e-5 <= alpha <= 1e-2


def test_round_bf16_definition():
    """RNE to bfloat16 (7 fraction bits): ties go to the even mantissa."""
    x = np.array([1.0, 1 + 2 ** -8, 1 + 3 * 2 ** -8, 1 + 2 ** -7, -(1 + 2 ** -8), 3.0, 0.0, 2 ** -130])
    want = np.array([1.0, 1.0, 1 + 2 ** -6, 1 + 2 ** -7, -1.0, 3.0, 0.0, 2 ** -130])
    assert np.array_equal(learn.round_bf16(x), want)
    r = np.random.default_rng(0).standard_normal(10000) * 10.0 ** np.random.default_rng(1).integers(-5, 5, 10000)
    q = learn.round_bf16(r)
    assert np.all(np.abs(q - r) <= 2.0 ** -8 * np.abs(r))          # within half a bf16 ulp (rel 2^-8)
    torch = pytest.importorskip("torch")
    assert np.array_equal(q, torch.from_numpy(r.astype(np.float32)).bfloat16().double().numpy())


def test_union_update_single_rank_is_ppo_update_and_union_gradient_is_rank_mean():
    """O-M: with W = 1 the union update is the single-rank update bit for bit; with W = 2 and
    identical rank batches and permutations, the union minibatch holds every row twice, so its mean-loss
    gradient and KL equal the single-rank ones, and the update equals ppo_update on one copy."""
    rng = np.random.default_rng(0)
    D, hid = 48, (32, 32, 32)
    T, N = 4, 24
    bt = synth.synthetic_storage(T, N, D, seed=5, p_term=0.1, p_timeout=0.05)
    theta = synth.init_params(D, hid, seed=2).astype(np.float64)
    perms = [rng.permutation(T * N) for _ in range(2)]
    z = np.zeros_like(theta)
    ref = learn.ppo_update(theta, z, z.copy(), 0, 1e-3, bt, perms, D, hid, n_epochs=2, n_minibatches=3)
    one = learn.ppo_update_union(theta, z, z.copy(), 0, 1e-3, [bt], [perms], D, hid, n_epochs=2, n_minibatches=3)
    assert np.array_equal(ref[0], one[0]) and ref[3] == one[3] and ref[4] == one[4]
    two = learn.ppo_update_union(theta, z, z.copy(), 0, 1e-3, [bt, bt], [perms, perms], D, hid, n_epochs=2,
                                 n_minibatches=3)
    # the duplicated union normalises with ddof = 1 over 2B samples instead of B: its std is smaller by
    # sqrt(2(B-1)/(2B-1)), so the two updates agree only to that O(1/B) difference
    assert two[3] == ref[3] and np.allclose(two[0], ref[0], rtol=0, atol=5e-4)
    A, _ = learn.gae(bt["r"], bt["V"], bt["V_T"], bt["b"], bt["term"], bt["timeout"])
    a = A.reshape(-1)
    s1, s2 = np.std(a, ddof=1), np.std(np.concatenate([a, a]), ddof=1)
    assert abs(s2 / s1 - np.sqrt(2.0 * (a.size - 1) / (2 * a.size - 1))) < 1e-12
