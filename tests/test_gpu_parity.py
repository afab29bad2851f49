"""GPU parity: the CUDA path (through the C ABI) against the independent oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): bit-exact for env state, resets, curriculum levels, indices and the
shuffle; |Δ| <= 1e-5·max(|ref|,1) for fp32 GAE/rewards/observations; bf16 MLP outputs and gradients
‖Δ‖/‖ref‖ <= 2e-2 (elementwise |Δ| <= 2e-2·(|ref| + rms(ref))); parameter drift after one PPO update
‖θ_gpu − θ_oracle‖/‖θ_oracle‖ <= 1e-3."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes only to be skipped
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle  # noqa: E402
from oracle import learn  # noqa: E402
import synth  # noqa: E402
from paper_2109_11978_b200 import lg  # noqa: E402
from paper_2109_11978_b200.context import Config, Context  # noqa: E402

ALL = lg.F_CURRICULUM | lg.F_NOISE | lg.F_PUSH | lg.F_BOOTSTRAP


def make(n_envs=256, T=8, hidden=(512, 256, 128), scan=(17, 11), levels=4, cols=5, flags=ALL, seed=11, K=4, E=5,
         rough=True):
    cfg = Config.make(n_envs=n_envs, n_steps=T, hidden=hidden, scan_nx=scan[0], scan_ny=scan[1], n_levels=levels,
                      n_cols=cols, flags=flags, seed=seed, n_minibatches=K, n_epochs=E)
    hf = synth.make_world(levels, cols, seed=3, rough=rough)
    ctx = Context(cfg, hf)
    theta = synth.init_params(cfg.obs_dim, hidden, seed=seed)
    ctx.params_set(theta)
    env = oracle.Env(n_envs, hf, levels, cols, seed=seed, scan=scan, flags=flags)
    return cfg, ctx, env, theta


def gpu_state(ctx):
    w = ctx.state_words.t().contiguous().cpu().numpy()
    return w.view(oracle.STATE_DTYPE).reshape(-1)


def set_gpu_state(ctx, st):
    w = np.ascontiguousarray(st).view(np.int32).reshape(len(st), 66)
    ctx.state_words.copy_(torch.from_numpy(np.ascontiguousarray(w.T)).cuda())
    torch.cuda.synchronize()


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def assert_bf16_close(a, ref, what="", ref_q=None, stats=None):
    """SURVEY §8(c).4 bf16 MLP outputs and gradients: ‖Δ‖/‖ref‖ <= 2e-2 per tensor against the exact fp64
    oracle AND elementwise |Δ| <= 2e-2·(|ref| + rms(ref)).  With ref_q (the oracle at the GPU's bf16 rounding
    points, DESIGN R28) the elementwise bound is applied against ref_q and the fraction of elements outside it
    against the exact oracle is reported in `stats`."""
    a = np.asarray(a, np.float64)
    ref = np.asarray(ref, np.float64)
    r = rel(a, ref)
    assert r <= 2e-2, (what, r)

    def worst_of(x, y):
        bound = 2e-2 * (np.abs(y) + np.sqrt(np.mean(y ** 2)))
        q = np.abs(x - y) / np.maximum(bound, 1e-300)
        return (float(np.max(q)) if q.size else 0.0), (float(np.mean(q > 1.0)) if q.size else 0.0)

    wx, fx = worst_of(a, ref)
    if ref_q is None:
        assert wx <= 1.0, (what, wx)
        return
    wq, _ = worst_of(a, np.asarray(ref_q, np.float64))
    if stats is not None:
        stats[what] = (r, wx, fx, wq)
    assert wq <= 1.0, (what, wq)


def per_tensor_drift(th, ref, D, hidden):
    """‖Δθ‖ / ‖θ_ref‖ per parameter tensor and overall."""
    pt = learn.unpack(np.asarray(th, np.float64) - ref, D, hidden)
    nr = np.linalg.norm(ref)
    return {k: np.linalg.norm(v) / nr for k, v in pt.items()}


def close_mixed(a, b, tol):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.all(np.abs(a - b) <= tol * np.maximum(np.abs(b), 1.0))


# ------------------------------------------------------------------ world generation (bit-exact)
@pytest.mark.parametrize("levels,cols,seed", [(10, 20, 0), (2, 7, (1 << 40) + 5), (1, 3, 9)])
def test_terrain_generate_bit_exact(levels, cols, seed):
    hf = torch.full((80 * levels, 80 * cols), float("nan"), device="cuda")
    lg.lg_terrain_generate(hf, levels, cols, seed)
    torch.cuda.synchronize()
    assert np.array_equal(hf.cpu().numpy(), oracle.terrain_generate(levels, cols, seed))


def test_terrain_world_runs_through_the_path():
    """A generated world serves as the env's heightfield: a short teacher-forced rollout stays bit-exact."""
    levels, cols = 4, 5
    hf_g = torch.empty((80 * levels, 80 * cols), device="cuda")
    lg.lg_terrain_generate(hf_g, levels, cols, 21)
    torch.cuda.synchronize()
    hf = hf_g.cpu().numpy()
    cfg = Config.make(n_envs=96, n_steps=8, scan_nx=17, scan_ny=11, n_levels=levels, n_cols=cols, flags=ALL, seed=4)
    ctx = Context(cfg, hf)
    ctx.params_set(synth.init_params(cfg.obs_dim, cfg.hidden, seed=4))
    env = oracle.Env(96, hf, levels, cols, seed=4, flags=ALL)
    obs_g = torch.zeros(96, cfg.obs_dim, device="cuda")
    ctx.reset(obs=obs_g)
    assert np.array_equal(obs_g.cpu().numpy(), env.reset())
    rng = np.random.default_rng(2)
    for t in range(8):
        a = (0.5 * rng.standard_normal((96, 12))).astype(np.float32)
        ctx.env_step(t, actions=torch.from_numpy(a).cuda(), obs=obs_g)
        o = env.step(a)[0]
        ctx.sync()
        assert np.array_equal(o, obs_g.cpu().numpy()), t
    assert gpu_state(ctx).tobytes() == env.state.tobytes()


# ------------------------------------------------------------------ environment (bit-exact)
@pytest.mark.parametrize("scan,rough,flags", [((17, 11), True, ALL), ((0, 0), False, ALL & ~lg.F_CURRICULUM)])
def test_env_teacher_forced_bit_exact(scan, rough, flags):
    cfg, ctx, env, _ = make(n_envs=200, T=24, scan=scan, rough=rough, flags=flags,
                            levels=4 if rough else 1, cols=5 if rough else 1)
    N, D = cfg.n_envs, cfg.obs_dim
    obs_g = torch.zeros(N, D, device="cuda")
    ctx.reset(obs=obs_g)
    o0 = env.reset()
    ctx.sync()
    assert gpu_state(ctx).tobytes() == env.state.tobytes()
    assert np.array_equal(obs_g.cpu().numpy(), o0)
    # force edge cases in both: time-outs, pushes, high levels at the top (loop-back), crashes
    st = env.state.copy()
    st["ep_step"][:20] = 998
    st["push_timer"][20:40] = 499
    if rough:
        st["level"][40:60] = 3
        st["crossed"][40:60] = 1
        st["ep_step"][40:60] = 999
    env.state[:] = st
    set_gpu_state(ctx, st)
    rng = np.random.default_rng(0)
    rew_g = torch.zeros(N, device="cuda")
    term_g = torch.zeros(N, dtype=torch.uint8, device="cuda")
    to_g = torch.zeros(N, dtype=torch.uint8, device="cuda")
    terms_g = torch.zeros(N, 9, device="cuda")
    n_to = n_term = 0
    for t in range(cfg.n_steps):
        a = (rng.standard_normal((N, 12)) * (0.3 + 1.5 * (t % 3 == 0))).astype(np.float32)
        a_g = torch.from_numpy(a).cuda()
        ctx.env_step(t, actions=a_g, obs=obs_g, reward=rew_g, terminated=term_g, timeout=to_g, terms=terms_g)
        o, r, te, to, terms, _ = env.step(a)
        ctx.sync()
        assert np.array_equal(te, term_g.cpu().numpy()), t
        assert np.array_equal(to, to_g.cpu().numpy()), t
        assert gpu_state(ctx).tobytes() == env.state.tobytes(), t
        assert np.array_equal(r, rew_g.cpu().numpy()), t
        assert np.array_equal(terms, terms_g.cpu().numpy()), t
        assert np.array_equal(o, obs_g.cpu().numpy()), t
        # the bf16 rollout row is the RNE rounding of the fp32 observation, pad columns zero
        row = ctx.obs[t + 1].float().cpu().numpy()
        assert np.array_equal(row[:, :D], torch.from_numpy(o).bfloat16().float().numpy())
        assert np.all(row[:, D:] == 0)
        n_to += int(to.sum())
        n_term += int(te.sum())
    assert n_to >= 20 and n_term > 0


def test_timeout_bootstrap_values_vs_oracle():
    """Time-out bootstrapping: the GPU compacts the pre-reset observation of every time-out
    of the rollout and evaluates the critic on all of them in one pass inside compute_gae; BOOT[t][i] must be
    the oracle critic on the oracle's pre-reset observation (bf16 rows, MLP tolerance) and 0 elsewhere."""
    cfg, ctx, env, theta = make(n_envs=256, T=12)
    N, D = cfg.n_envs, cfg.obs_dim
    ctx.reset()
    env.reset()
    ctx.sync()
    st = env.state.copy()
    st["ep_step"][:40] = 999 - (np.arange(40) % 6)  # time-outs spread over steps 0..5
    env.state[:] = st
    set_gpu_state(ctx, st)
    rng = np.random.default_rng(5)
    want = np.zeros((cfg.n_steps, N), np.float64)
    mask = np.zeros((cfg.n_steps, N), bool)
    for t in range(cfg.n_steps):
        a = (rng.standard_normal((N, 12)) * 0.3).astype(np.float32)
        ctx.env_step(t, actions=torch.from_numpy(a).cuda())
        _, _, te, to, _, tobs = env.step(a)
        idx = np.nonzero(to)[0]
        if idx.size:
            x = torch.from_numpy(tobs[idx]).bfloat16().float().numpy()
            _, v = _oracle_forward(theta, x.astype(np.float64), D, cfg.hidden)
            want[t, idx] = v
            mask[t, idx] = True
    assert mask.sum() >= 30
    ctx.compute_gae()
    ctx.sync()
    b = ctx.storage("BOOT").cpu().numpy()
    assert np.all(b[~mask] == 0.0)
    assert_bf16_close(b[mask], want[mask], "BOOT")
    assert int(ctx.scalars()["n_to_total"]) == int(mask.sum())


def test_curriculum_kernel_bit_exact():
    cfg, ctx, env, _ = make(n_envs=64, T=4, levels=10, cols=5)
    rng = np.random.default_rng(1)
    n = 5000
    crossed = (rng.random(n) < 0.4).astype(np.uint8)
    disp = rng.uniform(-12, 12, (n, 2)).astype(np.float32)
    cmd = rng.uniform(-1, 1, (n, 2)).astype(np.float32)
    ep = rng.integers(1, 1001, n).astype(np.int32)
    words = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    level = rng.integers(0, 10, n).astype(np.int32)
    lv_g = torch.from_numpy(level.copy()).cuda()
    ctx.curriculum(torch.from_numpy(crossed).cuda(), torch.from_numpy(disp).cuda(), torch.from_numpy(cmd).cuda(),
                   torch.from_numpy(ep).cuda(), torch.from_numpy(words.view(np.int32)).cuda(), lv_g)
    ctx.sync()
    want = [oracle.curriculum_level(int(level[i]), 10, int(crossed[i]), float(disp[i, 0]), float(disp[i, 1]),
                                    float(cmd[i, 0]), float(cmd[i, 1]), int(ep[i]), int(words[i])) for i in range(n)]
    assert np.array_equal(lv_g.cpu().numpy(), np.array(want, np.int32))


def test_shuffle_bit_exact():
    cfg, ctx, env, _ = make(n_envs=256, T=24, E=5)
    B = 256 * 24
    perm = torch.zeros(B, dtype=torch.int32, device="cuda")
    for e in range(5):
        ctx.shuffle(e, perm)
        ctx.sync()
        want = oracle.feistel_perm(B, oracle.shuffle_keys(cfg.seed, 0, 0, 5, e))
        assert np.array_equal(perm.cpu().numpy().view(np.uint32), want)


# ------------------------------------------------------------------ MLP (bf16 tolerance)
def _oracle_forward(theta, x, D, hidden):
    p = learn.unpack(theta.astype(np.float64), D, hidden)
    mu, _ = learn.mlp_forward(p, x, "a")
    v, _ = learn.mlp_forward(p, x, "c")
    return mu, v[:, 0]


@pytest.mark.parametrize("hidden,scan,M", [((512, 256, 128), (17, 11), 1000), ((128, 64, 32), (0, 0), 300),
                                           ((512, 256, 128), (0, 0), 4096)])
def test_policy_forward_vs_oracle(hidden, scan, M):
    cfg, ctx, env, theta = make(n_envs=max(M, 64), T=4, hidden=hidden, scan=scan, rough=scan[0] > 0,
                                levels=4 if scan[0] else 1, cols=5 if scan[0] else 1)
    rng = np.random.default_rng(2)
    x = np.zeros((M, cfg.obs_stride), np.float32)
    x[:, :cfg.obs_dim] = rng.standard_normal((M, cfg.obs_dim))
    xb = torch.from_numpy(x).cuda().bfloat16()
    mu = torch.zeros(M, 12, device="cuda")
    v = torch.zeros(M, device="cuda")
    ctx.forward(xb, mu, v)
    ctx.sync()
    mu_o, v_o = _oracle_forward(theta, xb.float().cpu().numpy()[:, :cfg.obs_dim], cfg.obs_dim, hidden)
    mg, vg = mu.cpu().numpy(), v.cpu().numpy()
    assert_bf16_close(mg, mu_o, "mu")
    assert_bf16_close(vg, v_o, "V")


def test_policy_act_rollout_vs_oracle():
    cfg, ctx, env, theta = make(n_envs=256, T=6)
    ctx.reset()
    env.reset()
    N = cfg.n_envs
    for t in range(cfg.n_steps):
        ctx.policy_act(t)
        ctx.sync()
        act = ctx.storage("ACT", extra=(12,))[t].cpu().numpy()
        mu = ctx.storage("MU", extra=(12,))[t].cpu().numpy()
        logp = ctx.storage("LOGP")[t].cpu().numpy()
        val = ctx.storage("VALUE")[t].cpu().numpy()
        x = ctx.obs[t].float().cpu().numpy()[:, :cfg.obs_dim]
        mu_o, v_o = _oracle_forward(theta, x, cfg.obs_dim, cfg.hidden)
        assert_bf16_close(mu, mu_o, "mu")
        assert_bf16_close(val, v_o, "V")
        eps = env.action_eps(s=t + 1)                         # Box-Muller noise is bit-defined
        assert np.max(np.abs((act - mu) - eps)) <= 4e-6 * np.max(np.abs(act) + 1)
        lp_o = learn.logp_gauss(act.astype(np.float64), mu.astype(np.float64), np.zeros(12))
        assert np.max(np.abs(logp - lp_o)) < 1e-4
        ctx.env_step(t)
        ctx.sync()
        o, *_ = env.step(act)
        assert gpu_state(ctx).tobytes() == env.state.tobytes()


@pytest.mark.parametrize("n_envs", [700, 4096])
def test_fused_policy_vs_per_layer_path(n_envs):
    """The fused rollout-policy kernel (three chained tcgen05 GEMMs + the head MMA + sampling in one CTA) against
    the per-layer GEMM + warp-per-row head path (LG_F_UNFUSED_POLICY), over a rollout (ragged last tile for
    700 envs). H3 is the same bits on both paths; the fused heads run on the tensor core (bf16 hi + lo head
    weights, shared with the update's loss epilogue) and the per-layer path's on the CUDA cores in fp32, so mu
    and V agree to fp32 level and the Box-Muller noise (act - mu) / sigma is the same draw. The rollouts are
    teacher-forced with the fused path's actions so the environment states stay identical."""
    outs = []
    acts = None
    for extra in (0, lg.F_UNFUSED_POLICY):
        cfg, ctx, env, theta = make(n_envs=n_envs, T=3, flags=ALL | extra)
        ctx.reset()
        res = {k: [] for k in ("ACT", "MU", "LOGP", "VALUE")}
        for t in range(cfg.n_steps):
            ctx.policy_act(t)
            ctx.sync()
            for k in res:
                res[k].append(ctx.storage(k, extra=(12,) if k in ("ACT", "MU") else ())[t].cpu().numpy().copy())
            if acts is None or len(acts) <= t:
                acts = (acts or []) + [res["ACT"][t]]
            ctx.env_step(t, actions=torch.from_numpy(acts[t]).cuda())
        ctx.sync()
        outs.append({k: np.stack(v) for k, v in res.items()})
    f, u = outs
    for k in ("MU", "VALUE"):
        scale = np.sqrt(np.mean(f[k].astype(np.float64) ** 2))
        assert np.max(np.abs(f[k] - u[k])) <= 1e-4 * scale, (k, float(np.max(np.abs(f[k] - u[k]))), scale)
    assert np.allclose(f["ACT"] - f["MU"], u["ACT"] - u["MU"], rtol=0, atol=1e-5)
    assert np.allclose(f["LOGP"], u["LOGP"], rtol=1e-6, atol=1e-4)


def test_first_minibatch_ratio_is_exactly_one():
    """The rollout's heads (k_policy_fused) and the update's loss epilogue evaluate mu with the same tensor-core
    instruction sequence on the same H3 bits, so on the first minibatch of an iteration (parameters unchanged
    since the rollout) mu_new == mu_old in every row: with log-std 0 the KL of every row is exactly 0, and the
    minibatch KL in the payload is exactly 0.0."""
    cfg, ctx, env, theta = make(n_envs=512, T=24, K=4)
    _rollout(ctx, cfg)
    ctx.compute_gae()
    B = cfg.n_envs * cfg.n_steps
    idx = np.random.default_rng(9).permutation(B)[:B // 4].astype(np.int32)
    ctx.minibatch_grad(torch.from_numpy(idx).cuda())
    ctx.sync()
    pay = ctx.grad[ctx.P:].cpu().numpy()
    assert pay[0] == 0.0 and pay[3] == 0.0, pay[:6]     # KL mean, clip fraction


def test_deterministic_policy_takes_the_mean_action():
    """LG_F_DETERMINISTIC (evaluation, NEXT-4): a = mu on both policy paths; the first step's mu equals the
    stochastic policy's (same weights, same reset), and logp is the density at the mean, -(sum ls + 6 ln 2pi)."""
    mus = []
    for extra in (lg.F_DETERMINISTIC, lg.F_DETERMINISTIC | lg.F_UNFUSED_POLICY, 0):
        cfg, ctx, env, theta = make(n_envs=300, T=2, flags=lg.F_NOISE | extra)
        ctx.reset()
        ctx.policy_act(0)
        ctx.sync()
        act = ctx.storage("ACT", extra=(12,))[0].cpu().numpy()
        mu = ctx.storage("MU", extra=(12,))[0].cpu().numpy()
        if extra:
            assert np.array_equal(act, mu)
            lp = ctx.storage("LOGP")[0].cpu().numpy()
            ls = theta[-12:].astype(np.float64)
            assert np.allclose(lp, -(ls.sum() + 6.0 * np.log(2.0 * np.pi)), rtol=1e-6, atol=1e-5)
        else:
            assert not np.array_equal(act, mu)
        mus.append(mu)
    assert mus[0].tobytes() == mus[2].tobytes()           # the fused path: deterministic and stochastic mu
    assert np.max(np.abs(mus[0] - mus[1])) <= 1e-4 * np.sqrt(np.mean(mus[0].astype(np.float64) ** 2))


def test_traversability_evaluation_vs_oracle():
    """NEXT-4 (P:119 Fig. caption): tools/evaluate.py's protocol -- robots spawned at the centre of every
    tile of a generated world (3 levels x 5 terrain kinds), command (0.75, U[-0.1, 0.1], 0), deterministic policy
    a = mu, no noise / pushes / curriculum -- replayed on the oracle environment with the GPU's actions: every
    robot's first outcome (tile exit before base contact / crash / neither) and its step are the same, the final
    environment state is bit-exact, and every step's actions equal the oracle MLP's mean on the same bf16
    observation rows within the bf16 tolerance."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "evaluate", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "evaluate.py"))
    ev = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ev)
    L, E, steps, seed = 3, 4, 150, 5
    ctx, hf, cmd = ev.setup(L, E, steps, seed)
    C = len(ev.KINDS)
    N = L * C * E
    env = oracle.Env(N, hf, L, C, seed=seed, flags=0)
    env.reset()
    k = np.arange(N) // E
    env.state["level"] = k // C
    env.state["col"] = k % C
    env.reset(init=False)
    env.state["cmd"] = cmd
    assert gpu_state(ctx).tobytes() == env.state.tobytes()
    out, stp, acts = ev.run(ctx, steps, record=True)
    theta = synth.init_params(ctx.cfg.obs_dim if hasattr(ctx.cfg, "obs_dim") else 235, (512, 256, 128), seed=seed)
    p = learn.unpack(theta.astype(np.float64), 235, (512, 256, 128))
    obs = ctx.obs.float().cpu().numpy()[:, :, :235]
    o_out = np.zeros(N, np.int8)
    o_stp = np.full(N, -1, np.int32)
    for t in range(steps):
        mu_o, _ = learn.mlp_forward(p, obs[t], "a")
        assert_bf16_close(acts[t], mu_o, f"mu t={t}")
        _, _, te, _, _, _ = env.step(acts[t])
        crashed = (te != 0) & (o_out == 0)
        crossed = (env.state["crossed"] != 0) & (o_out == 0) & ~crashed
        o_out[crashed] = -1
        o_out[crossed] = 1
        o_stp[crashed | crossed] = t + 1
    assert np.array_equal(out, o_out) and np.array_equal(stp, o_stp)
    assert gpu_state(ctx).tobytes() == env.state.tobytes()
    assert (o_out != 0).any()                          # the replay decides outcomes (crashes at least)


# ------------------------------------------------------------------ GAE (fp32 vs fp64 oracle)
def _rollout(ctx, cfg):
    ctx.reset()
    for t in range(cfg.n_steps):
        ctx.policy_act(t)
        ctx.env_step(t)
    ctx.sync()


def _batch_from_gpu(ctx, cfg):
    T, N = cfg.n_steps, cfg.n_envs
    flags = ctx.storage("FLAGS", torch.uint8).cpu().numpy()
    return dict(
        obs=ctx.obs[:T].float().cpu().numpy(),
        act=ctx.storage("ACT", extra=(12,)).cpu().numpy(), mu=ctx.storage("MU", extra=(12,)).cpu().numpy(),
        logp=ctx.storage("LOGP").cpu().numpy(), V=ctx.storage("VALUE").cpu().numpy(),
        r=ctx.storage("REWARD").cpu().numpy(), b=ctx.storage("BOOT").cpu().numpy(),
        term=(flags & 1), timeout=(flags >> 1) & 1,
        V_T=ctx.view("VALUE_T", torch.float32, (N,)).cpu().numpy(),
        logstd_old=ctx.theta[-12:].cpu().numpy())


def test_gae_vs_oracle_and_bootstrap_value():
    cfg, ctx, env, theta = make(n_envs=512, T=24)
    _rollout(ctx, cfg)
    # force some time-outs mid-rollout was done by the env (ep_step) only after 1000 steps; emulate via flags
    ctx.compute_gae()
    ctx.sync()
    bt = _batch_from_gpu(ctx, cfg)
    A_o, R_o = learn.gae(bt["r"], bt["V"], bt["V_T"], bt["b"], bt["term"], bt["timeout"])
    A = ctx.storage("ADV").cpu().numpy()
    R = ctx.storage("RET").cpu().numpy()
    assert close_mixed(A, A_o, 1e-5) and close_mixed(R, R_o, 1e-5)
    # V(o_T) is the critic on OBS slot T
    _, v_o = _oracle_forward(theta, ctx.obs[cfg.n_steps].float().cpu().numpy()[:, :cfg.obs_dim], cfg.obs_dim,
                             cfg.hidden)
    assert_bf16_close(bt["V_T"], v_o, "V_T")
    # the normalisation statistics (R13: whole batch, unbiased std) against the oracle's fp64 definition
    mean, inv_std = ctx.adv_normalization()
    assert abs(mean - A_o.mean()) <= 1e-6 * max(1.0, abs(A_o.mean()))
    assert abs(inv_std * (A_o.std(ddof=1) + 1e-8) - 1.0) <= 1e-6
    An = learn.normalize_adv(A_o)
    An_gpu = (A.astype(np.float64) - mean) * inv_std
    assert np.max(np.abs(An_gpu - An)) <= 1e-5 * max(1.0, np.max(np.abs(An)))


def test_gae_synthetic_flags_vs_oracle():
    cfg, ctx, env, theta = make(n_envs=300, T=16)
    ctx.reset()
    st = synth.synthetic_storage(cfg.n_steps, cfg.n_envs, cfg.obs_dim, seed=4, p_term=0.1, p_timeout=0.1)
    for name, key in (("REWARD", "r"), ("VALUE", "V"), ("BOOT", "b")):
        ctx.storage(name).copy_(torch.from_numpy(st[key]).cuda())
    ctx.storage("FLAGS", torch.uint8).copy_(torch.from_numpy((st["term"] | (st["timeout"] << 1)).astype(np.uint8)).cuda())
    torch.cuda.synchronize()
    ctx.compute_gae()
    ctx.sync()
    VT = ctx.view("VALUE_T", torch.float32, (cfg.n_envs,)).cpu().numpy()
    A_o, R_o = learn.gae(st["r"], st["V"], VT, st["b"], st["term"], st["timeout"])
    assert close_mixed(ctx.storage("ADV").cpu().numpy(), A_o, 1e-5)
    assert close_mixed(ctx.storage("RET").cpu().numpy(), R_o, 1e-5)


# ------------------------------------------------------------------ update (gradient and drift)
def _grad_tensors(g, D, hidden):
    return {k: v for k, v in learn.unpack(np.asarray(g, np.float64), D, hidden).items()}


# minibatch rows 3072 (dW split S = 6), 384 (S = 1: the tile written straight from shared memory),
# 600 (ragged 128-row tail), 12288 (S = 18, wide and narrow dW tiles)
@pytest.mark.parametrize("hidden,scan,N,T,K", [((512, 256, 128), (17, 11), 512, 24, 4),
                                               ((128, 64, 32), (0, 0), 64, 24, 4),
                                               ((512, 256, 128), (17, 11), 100, 24, 4),
                                               ((512, 256, 128), (17, 11), 1024, 24, 2),
                                               ((512, 256, 128), (0, 0), 512, 24, 4)])
def test_minibatch_gradient_vs_oracle(hidden, scan, N, T, K):
    cfg, ctx, env, theta = make(n_envs=N, T=T, hidden=hidden, scan=scan, rough=scan[0] > 0, K=K,
                                levels=4 if scan[0] else 1, cols=5 if scan[0] else 1)
    _rollout(ctx, cfg)
    ctx.compute_gae()
    ctx.sync()
    bt = _batch_from_gpu(ctx, cfg)
    B = N * T
    M = B // K
    idx = np.random.default_rng(5).permutation(B)[:M].astype(np.int32)
    ctx.minibatch_grad(torch.from_numpy(idx).cuda())
    ctx.sync()
    g_gpu = ctx.grad[:ctx.P].cpu().numpy()
    A_o, R_o = learn.gae(bt["r"], bt["V"], bt["V_T"], bt["b"], bt["term"], bt["timeout"])
    An = learn.normalize_adv(A_o).reshape(B)
    D = cfg.obs_dim
    obs = bt["obs"].reshape(B, -1)[:, :D]
    p = learn.unpack(theta.astype(np.float64), D, hidden)
    g_o, st = learn.ppo_minibatch(p, obs[idx], bt["act"].reshape(B, 12)[idx], bt["logp"].reshape(B)[idx],
                                  bt["V"].reshape(B)[idx], An[idx], R_o.reshape(B)[idx], bt["mu"].reshape(B, 12)[idx],
                                  bt["logstd_old"].astype(np.float64))
    g_q, _ = learn.ppo_minibatch(p, obs[idx], bt["act"].reshape(B, 12)[idx], bt["logp"].reshape(B)[idx],
                                 bt["V"].reshape(B)[idx], An[idx], R_o.reshape(B)[idx], bt["mu"].reshape(B, 12)[idx],
                                 bt["logstd_old"].astype(np.float64), quant="bf16")
    G = _grad_tensors(g_gpu, D, hidden)
    stats = {}
    for k, ref in g_o.items():
        assert_bf16_close(G[k], ref, k, ref_q=g_q[k], stats=stats)
    print("gradient parity (tensor: rel vs fp64, worst elementwise ratio vs fp64, fraction > 1 vs fp64, "
          "worst ratio vs bf16-point oracle): " +
          "; ".join(f"{k} {v[0]:.1e} {v[1]:.2f} {v[2]:.1e} {v[3]:.2f}" for k, v in stats.items()))
    assert max(v[2] for v in stats.values()) <= 1e-3      # vs fp64: at most 0.1 % of any tensor's elements
    pay = ctx.grad[ctx.P:].cpu().numpy()
    assert abs(pay[0] - st["kl"]) <= 2e-2 * max(abs(st["kl"]), 1e-4)
    assert abs(pay[2] - st["value_loss"]) <= 2e-2 * abs(st["value_loss"])


HEAD_KEYS = ("aW4", "ab4", "cW4", "cb4", "logstd")


@pytest.mark.parametrize("hidden,scan,N,T,K", [((512, 256, 128), (17, 11), 512, 24, 4),
                                               ((512, 256, 128), (17, 11), 100, 24, 4),
                                               ((128, 64, 32), (0, 0), 64, 24, 4),
                                               ((512, 256, 128), (17, 11), 4096, 24, 4)])
def test_fused_loss_epilogue_vs_two_kernel_path(hidden, scan, N, T, K):
    """The PPO loss head fused into the layer-3 GEMM's epilogue (default) against the layer-3 GEMM + warp-per-row
    loss kernel (LG_F_UNFUSED_LOSS). The fused path forms mu / V, dH3 = dmu W4 and dW4 = H3^T dmu on the tensor
    cores from three-part bf16 splits of the fp32 operands (exact operands, another summation order) where the
    two-kernel path runs fp32 FMA chains, and the per-row loss terms are the same expressions (common.cuh), so:
    the head gradients (W4, b4, log-std) agree to fp32 level (elementwise <= 1e-4 (|ref| + rms)); dZ3 may differ
    by one bf16 ulp in rare elements, which propagates through the bf16 rounding points of dZ2 / dZ1 (DESIGN R28),
    so the lower layers' gradients are held to the north_star bf16 bound between the two paths; the loss
    statistics agree to 1e-5. Ragged tail (600 rows), the flat C1 net (H2 = 32 inside a 128-wide tile) and the
    full C3 minibatch (24,576 rows)."""
    B = N * T
    idx = np.random.default_rng(5).permutation(B)[:B // K].astype(np.int32)
    res = []
    for extra in (0, lg.F_UNFUSED_LOSS):
        cfg, ctx, env, theta = make(n_envs=N, T=T, hidden=hidden, scan=scan, rough=scan[0] > 0, K=K,
                                    levels=4 if scan[0] else 1, cols=5 if scan[0] else 1, flags=ALL | extra)
        _rollout(ctx, cfg)
        ctx.compute_gae()
        ctx.minibatch_grad(torch.from_numpy(idx).cuda())
        ctx.sync()
        res.append((ctx.grad[:ctx.P].cpu().numpy().copy(), ctx.grad[ctx.P:].cpu().numpy().copy()))
    D = cfg.obs_dim
    gf, gu = _grad_tensors(res[0][0], D, hidden), _grad_tensors(res[1][0], D, hidden)
    worst = {}
    for k in gf:
        a, b = gf[k], gu[k]
        f = 1e-4 if k in HEAD_KEYS else 2e-2
        tol = f * (np.abs(b) + np.sqrt(np.mean(b ** 2))) + 1e-30
        worst[k] = (rel(a, b), float(np.max(np.abs(a - b) / tol)))
        assert worst[k][1] <= 1.0 and worst[k][0] <= (1e-5 if k in HEAD_KEYS else 2e-3), (k, worst[k])
    print("fused vs two-kernel loss (rel, worst elementwise ratio): " +
          " ".join(f"{k}:{v[0]:.1e}/{v[1]:.2f}" for k, v in worst.items()))
    pf, pu = res[0][1], res[1][1]
    # KL, surrogate, value loss, clip fraction: the fused path's mu / V are the rollout's bits (tensor-core heads),
    # the two-kernel path's are the CUDA-core fp32 heads (same operands, another summation order), so the ratio
    # of the first minibatch is exactly 1 on the fused path and 1 +- ~1e-7 on the other
    assert abs(pf[0] - pu[0]) <= 1e-9 and pf[3] == pu[3], (pf[:4], pu[:4])
    for i in (1, 2):
        assert abs(pf[i] - pu[i]) <= 1e-5 * abs(pu[i]), (i, pf[i], pu[i])
    assert pf[4] == pu[4] == 0.0 and pf[5] == pu[5] == 1.0


@pytest.mark.parametrize("scan,rough", [((17, 11), True), ((0, 0), False)])
def test_ppo_update_parameter_drift_vs_oracle(scan, rough):
    """One complete update (5 x 4 minibatches) against the oracle, rough (C3 network) and flat (C2 network).
    DESIGN R28: the north_star bound (drift <= 1e-3) holds against the oracle evaluated at the GPU's bf16
    operand rounding points (SURVEY §8(c).1's switch); against the exact fp64 oracle the GPU may drift by no
    more than the oracle's own bf16-vs-fp64 gap plus 1e-3 (tools/drift_precision.py: bf16 rounding at any one
    point alone moves an Adam update by ~2e-3)."""
    cfg, ctx, env, theta = make(n_envs=512, T=24, scan=scan, rough=rough, levels=4 if rough else 1,
                                cols=5 if rough else 1)
    _rollout(ctx, cfg)
    ctx.compute_gae()
    ctx.sync()
    bt = _batch_from_gpu(ctx, cfg)
    B = cfg.n_envs * cfg.n_steps
    perms = []
    pt = torch.zeros(B, dtype=torch.int32, device="cuda")
    for e in range(cfg.n_epochs):
        ctx.shuffle(e, pt)
        ctx.sync()
        perms.append(pt.cpu().numpy().view(np.uint32).copy())
    stats = torch.zeros(64, dtype=torch.int32, device="cuda")
    ctx.update(stats)
    ctx.sync()
    th_gpu = ctx.theta.cpu().numpy().astype(np.float64)
    z = np.zeros(theta.size)
    th_q, m, v, t, alpha, st = learn.ppo_update(theta.astype(np.float64), z, z.copy(), 0, 1e-3, bt, perms,
                                                cfg.obs_dim, cfg.hidden, quant="bf16")
    th_x, *_ = learn.ppo_update(theta.astype(np.float64), z, z.copy(), 0, 1e-3, bt, perms, cfg.obs_dim, cfg.hidden)
    sc = ctx.scalars()
    assert sc["adam_t"] == t == 20
    assert abs(sc["alpha"] - alpha) <= 1e-6 * alpha
    drift_q, drift_x, gap = rel(th_gpu, th_q), rel(th_gpu, th_x), rel(th_q, th_x)
    per = per_tensor_drift(th_gpu, th_x, cfg.obs_dim, cfg.hidden)
    print(f"drift vs bf16-point oracle {drift_q:.3e}; vs exact fp64 oracle {drift_x:.3e} (oracle gap {gap:.3e}); "
          f"update size {rel(th_x, theta):.3e}; per tensor vs fp64: " +
          " ".join(f"{k}:{v:.1e}" for k, v in sorted(per.items(), key=lambda kv: -kv[1])[:6]))
    assert drift_q <= 1e-3
    assert drift_x <= gap + 1e-3
    for k, d in per_tensor_drift(th_gpu, th_q, cfg.obs_dim, cfg.hidden).items():
        assert d <= 1e-3, k


def test_update_with_adam_summing_dw_partials_is_bit_identical():
    """Single-rank ppo_update lets the weight-gradient GEMMs store only their split-K partials and Adam sum them
    in split order (no grid barrier / reduction pass): the same sums as the GEMMs' own reductions, so θ after two
    iterations is bit-identical with every reduction in the GEMMs (LG_DW1_PARTIAL=0 LG_DW23_PARTIAL=0) and with
    only layer 1's in Adam (separate processes: the switches are read once per process)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, %r)\n"
        "import synth\n"
        "from paper_2109_11978_b200.context import Config, Context\n"
        "cfg = Config.make(n_envs=512, n_steps=24, scan_nx=17, scan_ny=11, n_levels=4, n_cols=5, flags=15, seed=4)\n"
        "ctx = Context(cfg, synth.make_world(4, 5, seed=3, rough=True))\n"
        "ctx.params_set(synth.init_params(cfg.obs_dim, cfg.hidden, seed=4))\n"
        "ctx.reset()\n"
        "for _ in range(2): ctx.iteration()\n"
        "ctx.sync()\n"
        "sys.stdout.buffer.write(ctx.theta.cpu().numpy().tobytes())\n") % root
    outs = []
    for v1, v23 in (("1", "1"), ("0", "0"), ("1", "0")):  # default (all in Adam), all in the GEMMs, layer 1 only
        env = dict(os.environ, LG_DW1_PARTIAL=v1, LG_DW23_PARTIAL=v23)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, env=env, timeout=300)
        assert r.returncode == 0, r.stderr.decode()[-2000:]
        outs.append(r.stdout)
    assert len(outs[0]) > 0 and outs[0] == outs[1] == outs[2]


# ------------------------------------------------------------------ whole iteration, graph replay
@pytest.mark.parametrize("n_envs,T,levels,cols", [(256, 8, 4, 5), (4096, 24, 10, 20), (16384, 50, 10, 20)])
def test_iteration_graph_replay_matches_eager(n_envs, T, levels, cols):
    """The launch configuration bench.py times (one CUDA graph per iteration, dW on the second stream) gives
    the same bits as the eager C-ABI calls, at a small size, at the full C3 size (4096 x 24) and at the
    sweep's largest batch (16384 x 50)."""
    cfgs = []
    for mode in ("eager", "graph"):
        cfg, ctx, env, theta = make(n_envs=n_envs, T=T, seed=21, levels=levels, cols=cols)
        ctx.reset()
        if mode == "eager":
            for _ in range(3):
                ctx.iteration()
        else:
            ctx.capture()
            for _ in range(3):
                ctx.replay()
        ctx.sync()
        cfgs.append((ctx.theta.cpu().numpy().copy(), gpu_state(ctx).tobytes(), ctx.scalars()))
    assert np.array_equal(cfgs[0][0], cfgs[1][0])
    assert cfgs[0][1] == cfgs[1][1]
    assert cfgs[0][2]["iteration"] == 3 and cfgs[1][2]["iteration"] == 3


def test_iterate_host_stats_finite():
    cfg, ctx, env, theta = make(n_envs=512, T=24)
    ctx.reset()
    s = ctx.iterate_host()
    d = s.as_dict()
    assert d["minibatches_applied"] == 20 and d["nonfinite_skips"] == 0
    for k in ("surrogate_loss", "value_loss", "entropy", "mean_kl", "lr"):
        assert np.isfinite(d[k])
    assert np.float32(1e-5) <= d["lr"] <= np.float32(1e-2)
    assert sum(d["level_hist"]) == cfg.n_envs


# ------------------------------------------------------------------ checkpoint / resume, ablation arms
def test_checkpoint_resume_bit_exact():
    """lg_resume: a run restored from a checkpoint continues bit-identically."""
    cfg, ctx, env, theta = make(n_envs=256, T=8, seed=9)
    ctx.reset()
    ctx.capture()
    for _ in range(2):
        ctx.replay()
    ck = ctx.checkpoint()
    for _ in range(3):
        ctx.replay()
    ctx.sync()
    names = ("THETA", "ADAM_M", "ADAM_V", "STATE", "OBS", "ADV", "RET")
    ref = {k: ctx.bufs[lg.BUF[k]].cpu() for k in names}
    sc_ref = ctx.scalars()
    hf = synth.make_world(4, 5, seed=3, rough=True)
    ctx2 = Context(cfg, hf)
    ctx2.restore(ck)
    ctx2.capture()
    for _ in range(3):
        ctx2.replay()
    ctx2.sync()
    for k in names:
        assert torch.equal(ctx2.bufs[lg.BUF[k]].cpu(), ref[k]), k
    assert ctx2.scalars() == sc_ref
    bad = dict(ck, config=dict(ck["config"], n_steps=9))
    with pytest.raises(ValueError):
        ctx2.restore(bad)


def test_bootstrap_arms_identical_until_a_timeout():
    """NEXT-1 pin (time-out bootstrapping): the bootstrap-on and -off arms of a paired run are
    bit-identical while no episode times out, and differ in θ once time-outs occur (episode step 1000)."""
    res = {}
    for arm, fl in (("on", ALL), ("off", ALL & ~lg.F_BOOTSTRAP)):
        cfg, ctx, env, theta = make(n_envs=256, T=8, seed=5, flags=fl)
        ctx.reset()
        ctx.capture()
        for _ in range(2):
            ctx.replay()
        ctx.sync()
        before = ctx.theta.cpu().numpy().copy()
        st = gpu_state(ctx)
        st["ep_step"][:96] = 995  # these episodes reach 1000 steps (time-out) at step 4 of the next iteration
        set_gpu_state(ctx, st)
        ctx.replay()
        ctx.sync()
        res[arm] = (before, ctx.theta.cpu().numpy().copy(), ctx.scalars(), gpu_state(ctx).tobytes())
    assert np.array_equal(res["on"][0], res["off"][0])
    assert res["on"][2]["n_to_total"] > 0 and res["off"][2]["n_to_total"] == 0
    assert res["on"][3] == res["off"][3]                 # the environment does not depend on the flag
    assert not np.array_equal(res["on"][1], res["off"][1])


# ------------------------------------------------------------------ BASELINE configs[2] full size (C3)
def test_env_full_size_c3_bit_exact():
    """4096 envs x 24 steps on the C3 world (10 levels x 20 columns, 187-point scan, curriculum, noise, pushes),
    teacher-forced with random actions: state, observation, reward and flags bit-exact at every step, in the
    launch configuration bench.py times (same kernels, same grid shapes)."""
    cfg, ctx, env, _ = make(n_envs=4096, T=24, levels=10, cols=20, seed=1234)
    N = cfg.n_envs
    obs_g = torch.zeros(N, cfg.obs_dim, device="cuda")
    ctx.reset(obs=obs_g)
    o0 = env.reset()
    ctx.sync()
    assert gpu_state(ctx).tobytes() == env.state.tobytes() and np.array_equal(obs_g.cpu().numpy(), o0)
    st = env.state.copy()
    st["ep_step"][::97] = 990        # time-outs during the rollout
    st["push_timer"][1::53] = 495    # pushes
    st["level"][2::41] = 9           # top-level promotions loop back
    st["crossed"][2::41] = 1
    st["ep_step"][2::41] = 995
    env.state[:] = st
    set_gpu_state(ctx, st)
    rng = np.random.default_rng(3)
    rew_g = torch.zeros(N, device="cuda")
    term_g = torch.zeros(N, dtype=torch.uint8, device="cuda")
    to_g = torch.zeros(N, dtype=torch.uint8, device="cuda")
    n_to = 0
    for t in range(cfg.n_steps):
        a = (rng.standard_normal((N, 12)) * 0.5).astype(np.float32)
        ctx.env_step(t, actions=torch.from_numpy(a).cuda(), obs=obs_g, reward=rew_g, terminated=term_g, timeout=to_g)
        o, r, te, to, _, _ = env.step(a)
        ctx.sync()
        assert gpu_state(ctx).tobytes() == env.state.tobytes(), t
        assert np.array_equal(o, obs_g.cpu().numpy()), t
        assert np.array_equal(r, rew_g.cpu().numpy()), t
        assert np.array_equal(te, term_g.cpu().numpy()) and np.array_equal(to, to_g.cpu().numpy()), t
        n_to += int(to.sum())
    assert n_to >= 40


def test_rollout_gae_and_minibatch_gradient_full_size_c3():
    """The full C3 rollout through the GPU path (fused policy, env kernels), GAE with time-out bootstrap over
    98,304 samples against the oracle (1e-5), and one full-size minibatch (M = 24,576) gradient against the
    fp64 oracle (bf16 MLP tolerance 2e-2)."""
    cfg, ctx, env, theta = make(n_envs=4096, T=24, levels=10, cols=20, seed=1234)
    ctx.reset()
    st = gpu_state(ctx)
    st["ep_step"][::61] = 990         # time-outs inside the rollout exercise the bootstrap path
    set_gpu_state(ctx, st)
    for t in range(cfg.n_steps):
        ctx.policy_act(t)
        ctx.env_step(t)
    ctx.compute_gae()
    ctx.sync()
    bt = _batch_from_gpu(ctx, cfg)
    assert bt["timeout"].sum() >= 60
    A_o, R_o = learn.gae(bt["r"], bt["V"], bt["V_T"], bt["b"], bt["term"], bt["timeout"])
    assert close_mixed(ctx.storage("ADV").cpu().numpy(), A_o, 1e-5)
    assert close_mixed(ctx.storage("RET").cpu().numpy(), R_o, 1e-5)
    # bootstrap values: the critic on the pre-reset observation of every time-out
    to_idx = np.argwhere(bt["timeout"] > 0)
    assert np.all(bt["b"][bt["timeout"] == 0] == 0.0)
    B = cfg.n_envs * cfg.n_steps
    M = B // cfg.n_minibatches
    idx = np.random.default_rng(11).permutation(B)[:M].astype(np.int32)
    ctx.minibatch_grad(torch.from_numpy(idx).cuda())
    ctx.sync()
    g_gpu = ctx.grad[:ctx.P].cpu().numpy()
    An = learn.normalize_adv(A_o).reshape(B)
    D = cfg.obs_dim
    obs = bt["obs"].reshape(B, -1)[:, :D]
    p = learn.unpack(theta.astype(np.float64), D, cfg.hidden)
    g_o, _ = learn.ppo_minibatch(p, obs[idx], bt["act"].reshape(B, 12)[idx], bt["logp"].reshape(B)[idx],
                                 bt["V"].reshape(B)[idx], An[idx], R_o.reshape(B)[idx], bt["mu"].reshape(B, 12)[idx],
                                 bt["logstd_old"].astype(np.float64))
    g_q, _ = learn.ppo_minibatch(p, obs[idx], bt["act"].reshape(B, 12)[idx], bt["logp"].reshape(B)[idx],
                                 bt["V"].reshape(B)[idx], An[idx], R_o.reshape(B)[idx], bt["mu"].reshape(B, 12)[idx],
                                 bt["logstd_old"].astype(np.float64), quant="bf16")
    G = _grad_tensors(g_gpu, D, cfg.hidden)
    stats = {}
    for k, ref in g_o.items():
        assert_bf16_close(G[k], ref, k, ref_q=g_q[k], stats=stats)
    print("C3 gradient parity (tensor: rel vs fp64, worst elementwise ratio vs fp64, fraction > 1 vs fp64, "
          "worst ratio vs bf16-point oracle): " +
          "; ".join(f"{k} {v[0]:.1e} {v[1]:.2f} {v[2]:.1e} {v[3]:.2f}" for k, v in stats.items()))
    assert max(v[2] for v in stats.values()) <= 1e-3
    assert len(to_idx) == int(bt["timeout"].sum())


def test_ppo_update_drift_full_size_c3():
    """All 5 x 4 minibatches of one C3 iteration (M = 24,576): parameter drift after the update against the
    oracle with the GPU's bf16 rounding points <= 1e-3 relative (BASELINE north_star), against the exact fp64
    oracle <= the oracle's own rounding-point gap + 1e-3 (DESIGN R28); Alg. 1 state equal."""
    cfg, ctx, env, theta = make(n_envs=4096, T=24, levels=10, cols=20, seed=1234)
    _rollout(ctx, cfg)
    ctx.compute_gae()
    ctx.sync()
    bt = _batch_from_gpu(ctx, cfg)
    B = cfg.n_envs * cfg.n_steps
    perms = []
    pt = torch.zeros(B, dtype=torch.int32, device="cuda")
    for e in range(cfg.n_epochs):
        ctx.shuffle(e, pt)
        ctx.sync()
        perms.append(pt.cpu().numpy().view(np.uint32).copy())
    stats = torch.zeros(64, dtype=torch.int32, device="cuda")
    ctx.update(stats)
    ctx.sync()
    th_gpu = ctx.theta.cpu().numpy().astype(np.float64)
    z = np.zeros(theta.size)
    th_q, m, v, t, alpha, st = learn.ppo_update(theta.astype(np.float64), z, z.copy(), 0, 1e-3, bt, perms,
                                                cfg.obs_dim, cfg.hidden, quant="bf16")
    th_x, *_ = learn.ppo_update(theta.astype(np.float64), z, z.copy(), 0, 1e-3, bt, perms, cfg.obs_dim, cfg.hidden)
    sc = ctx.scalars()
    assert sc["adam_t"] == t == 20
    assert abs(sc["alpha"] - alpha) <= 1e-6 * alpha
    drift_q, drift_x, gap = rel(th_gpu, th_q), rel(th_gpu, th_x), rel(th_q, th_x)
    print(f"C3 drift vs bf16-point oracle {drift_q:.3e}; vs exact fp64 oracle {drift_x:.3e} (oracle gap {gap:.3e})")
    assert drift_q <= 1e-3
    assert drift_x <= gap + 1e-3                          # DESIGN R28
