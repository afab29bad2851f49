"""Pins for the environment side of the oracle (oracle/env_oracle.c) against what the paper, SPEC and
mathematics fix -- never against the oracle itself.  CPU only."""
import math
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


# ---------------------------------------------------------------- Philox
def test_philox_known_answers():
    for r in _rows("philox_kat.txt"):
        v = [int(x, 16) for x in r]
        out = oracle.philox(v[0], v[1], v[2:6])
        assert list(out) == v[6:10]


# ---------------------------------------------------------------- polynomials
def test_sincos_matches_libm():
    x = np.linspace(-12.0, 12.0, 20001).astype(np.float32)
    s, c = oracle.sincos(x)
    xd = x.astype(np.float64)
    assert np.max(np.abs(s - np.sin(xd))) < 3e-7
    assert np.max(np.abs(c - np.cos(xd))) < 3e-7
    s0, c0 = oracle.sincos(np.zeros(1, np.float32))
    assert s0[0] == 0.0 and c0[0] == 1.0


def test_exp_log_match_libm():
    x = np.linspace(-30.0, 30.0, 20001).astype(np.float32)
    y = oracle.exp(x)
    assert np.max(np.abs(y / np.exp(x.astype(np.float64)) - 1.0)) < 4e-7
    assert oracle.exp(np.zeros(1, np.float32))[0] == 1.0
    u = np.geomspace(2.0 ** -24, 1.0, 20001).astype(np.float32)
    lg = oracle.log(u)
    assert np.max(np.abs(lg - np.log(u.astype(np.float64)))) < 4e-6
    assert oracle.log(np.ones(1, np.float32))[0] == 0.0


# ---------------------------------------------------------------- height lookups
HF22 = np.array([[0.0, 2.0], [1.0, 4.0]], np.float32)  # hf[i][j], i along x


def test_plate_hand_grid():
    assert oracle.h_plate(HF22, 0.0625, 0.125) == 2.0          # cell (0, 1)
    assert oracle.h_plate(HF22, 0.15, 0.05) == 1.0
    x = float(np.float32(0.1))                                  # 0.1f*10 == 1.0f: lower index owns
    assert oracle.h_plate(HF22, x, 0.05) == 0.0
    xn = float(np.nextafter(np.float32(0.1), np.float32(1.0)))
    assert oracle.h_plate(HF22, xn, 0.05) == 1.0
    assert oracle.h_plate(HF22, -5.0, 9.0) == 2.0               # clamped to the border cell
    flat = np.zeros((80, 80), np.float32)
    assert oracle.h_plate(flat, 3.3, 7.7) == 0.0


def test_plate_riser_straddle():
    # stairs tile: two points 0.05 m apart straddling a riser differ by exactly the riser
    hf = synth.generate_tile(4, 9, 10, seed=0)
    i = next(k for k in range(79) if hf[k + 1, 40] != hf[k, 40])
    x_lo, x_hi = (i + 0.75) * 0.1, (i + 1.25) * 0.1
    d = oracle.h_plate(hf, x_hi, 4.05) - oracle.h_plate(hf, x_lo, 4.05)
    assert abs(d - np.float32(0.2)) < 1e-6


def test_bilinear_hand_grid():
    assert oracle.h_bilinear(HF22, 0.0625, 0.125) == 1.71875
    assert oracle.h_bilinear(HF22, 0.05, 0.05) == 0.0           # node = cell centre
    assert oracle.h_bilinear(HF22, 0.15, 0.15) == 4.0
    assert oracle.h_bilinear(HF22, 0.2, 0.2) == 4.0             # clamped at the border
    assert oracle.h_bilinear(HF22, 0.1, 0.05) == 0.5


def test_bilinear_reproduces_linear_ramp_and_plates():
    i = np.arange(20, dtype=np.float32)[:, None]
    j = np.arange(30, dtype=np.float32)[None, :]
    hf = (0.25 * i + 0.5 * j).astype(np.float32)               # exactly representable plane
    rng = np.random.default_rng(1)
    for _ in range(200):
        fx, fy = rng.integers(0, 19 * 8) / 8.0, rng.integers(0, 29 * 8) / 8.0   # dyadic node offsets
        x, y = (fx + 0.5) / 10.0, (fy + 0.5) / 10.0
        got = oracle.h_bilinear(hf, np.float32(x), np.float32(y))
        assert abs(got - (0.25 * fx + 0.5 * fy)) < 1e-5
    hf2 = np.full((4, 4), 0.7, np.float32)
    assert abs(oracle.h_bilinear(hf2, 0.17, 0.23) - np.float32(0.7)) < 1e-7


# ---------------------------------------------------------------- kinematics
def test_fk_straight_leg_and_default_pose():
    for leg in range(4):
        p, _ = oracle.leg_fk(leg, [0.0, 0.0, 0.0])
        hip = np.array([[0.3, 0.15], [0.3, -0.15], [-0.3, 0.15], [-0.3, -0.15]][leg])
        assert abs(p[2] - (-0.7)) < 1e-6                       # l_thigh + l_shank
        assert abs(p[0] - hip[0]) < 1e-6
    zs = [oracle.leg_fk(l, QDEF[3 * l:3 * l + 3])[0][2] for l in range(4)]
    assert max(zs) == min(zs)                                   # all feet at identical z
    assert abs(zs[0] + 0.7 * math.cos(0.7)) < 1e-6


def test_fk_jacobian_vs_finite_differences():
    rng = np.random.default_rng(0)
    for _ in range(20):
        leg = int(rng.integers(0, 4))
        q = rng.uniform(-1.0, 1.0, 3)
        _, J = oracle.leg_fk(leg, q)
        h = 1e-2
        for k in range(3):
            dq = np.zeros(3)
            dq[k] = h
            pp, _ = oracle.leg_fk(leg, q + dq)
            pm, _ = oracle.leg_fk(leg, q - dq)
            fd = (pp.astype(np.float64) - pm) / (2 * h)
            assert np.max(np.abs(fd - J[k])) < 2e-4


def _env(n=1, rough=False, flags=0, scan=(17, 11)):
    hf = synth.make_world(1, 1, rough=False) if not rough else synth.make_world(10, 20, seed=0)
    nl, nc = (1, 1) if not rough else (10, 20)
    return oracle.Env(n, hf, nl, nc, seed=123, scan=scan, flags=flags)


QDEF = np.array([0, 0.7, -1.4, 0, 0.7, -1.4, 0, -0.7, 1.4, 0, -0.7, 1.4], np.float32)


def _place(env, i, z, q=None):
    st = env.state
    st["p"][i] = (4.0, 4.0, z)
    st["quat"][i] = (1.0, 0.0, 0.0, 0.0)
    st["v"][i] = 0.0
    st["w"][i] = 0.0
    st["q"][i] = QDEF if q is None else q
    st["qd"][i] = 0.0
    st["aprev"][i] = 0.0
    st["mu"][i] = 1.0
    st["contact"][i] = 0
    st["tair"][i] = 0.0


# ---------------------------------------------------------------- PD / free fall
def test_pd_torque_examples_and_free_fall():
    env = _env()
    env.reset()
    _place(env, 0, 5.0)
    a = np.zeros(12, np.float32)
    tau, qdd, airsum, crash, nc, fz = env.transition_single(0, a)
    assert np.all(tau == 0.0) and np.all(qdd == 0.0)            # q = q*, q̇ = 0 -> τ = 0
    assert fz == 0.0 and crash == 0
    vz = env.state["v"][0][2]
    assert abs(vz - (-4 * 9.81 * 0.005)) < 1e-6                 # 4 substeps of Δv_z = −0.04905
    assert np.all(env.state["v"][0][:2] == 0.0)
    # saturation: q* - q = 10 -> τ = τ_max = 80 exactly
    _place(env, 0, 5.0)
    a = np.zeros(12, np.float32)
    a[4] = 20.0
    tau, *_ = env.transition_single(0, a)
    assert tau[4] == 80.0


def test_contact_force_examples():
    c, f = oracle.contact_force(0.0, [0, 0, -0.01], [0, 0, 0], 1.0)      # δ = 0.01 -> 50 N
    assert c == 1 and abs(f[2] - 50.0) < 1e-4 and f[0] == 0.0 and f[1] == 0.0
    c, f = oracle.contact_force(0.0, [0, 0, 0.02], [0, 0, 0], 1.0)       # above ground -> 0
    assert c == 0 and np.all(f == 0.0)
    c, f = oracle.contact_force(0.0, [0, 0, -0.02], [10.0, 0, 0], 0.5)   # Coulomb cap 0.5·100
    assert abs(f[2] - 100.0) < 1e-3 and abs(abs(f[0]) - 50.0) < 1e-3 and f[0] < 0
    c, f = oracle.contact_force(0.0, [0, 0, -0.02], [0.1, 0.0, 0], 0.5)  # below the cap: c_t·|v_t|
    assert abs(f[0] + 60.0 * 0.1) < 1e-4
    c, f = oracle.contact_force(0.0, [0, 0, -0.01], [0, 0, 1.0], 1.0)    # damping cannot pull
    assert f[2] == 0.0


def test_standing_settles_to_weight():
    # default pose on flat ground -> Σ f_n → m·g within 2 % after 1 s of settling
    env = _env()
    env.reset()
    _place(env, 0, 0.5354 - 0.002)
    a = np.zeros(12, np.float32)
    fz_hist = []
    for _ in range(100):
        *_, fz = env.transition_single(0, a)
        fz_hist.append(fz)
    assert abs(np.mean(fz_hist[50:]) - 30.0 * 9.81) / (30.0 * 9.81) < 0.02   # window after 1 s
    assert abs(fz_hist[-1] - 30.0 * 9.81) / (30.0 * 9.81) < 0.02
    q = env.state["quat"][0]
    assert abs(np.sum(q.astype(np.float64) ** 2) - 1.0) < 1e-6


def test_quaternion_norm_long_run_and_yaw_equivariance():
    env = _env(n=2)
    env.reset()
    rng = np.random.default_rng(0)
    for i in range(2):
        _place(env, i, 3.0)
    env.state["w"][0] = (0.3, -0.2, 0.5)
    psi = np.float32(math.pi / 2)
    sh, ch = math.sin(psi / 2), math.cos(psi / 2)
    env.state["w"][1] = (0.3, -0.2, 0.5)
    env.state["quat"][1] = (ch, 0, 0, sh)
    for _ in range(500):
        env.transition_single(0, np.zeros(12, np.float32))
    qn = env.state["quat"][0].astype(np.float64)
    assert abs(np.sum(qn ** 2) - 1.0) < 1e-6


# ---------------------------------------------------------------- reward (Table 2)
def _rec(v=(0, 0, 0), w=(0, 0, 0), cmd=(0, 0, 0)):
    r = np.zeros(1, oracle.STATE_DTYPE)[0]
    r["quat"] = (1, 0, 0, 0)
    r["v"] = v
    r["w"] = w
    r["cmd"] = cmd
    return r


def test_reward_examples():
    gold = {row[0]: (int(row[1]), float(row[2])) for row in _rows("reward_examples.txt")}
    z12 = np.zeros(12, np.float32)
    terms, tot = oracle.reward_terms(_rec(v=(0.7, -0.2, 0), w=(0, 0, 0.3), cmd=(0.7, -0.2, 0.3)), z12, z12, z12, 0.0, 0)
    k, val = gold["perfect_tracking"]
    assert abs(terms[k] - val) < 1e-6 and abs(terms[1] - 0.01) < 1e-6
    assert np.all(terms[2:] == 0.0)
    assert abs(tot - np.sum(terms.astype(np.float64))) < 1e-6   # breakdown sums to total
    terms, _ = oracle.reward_terms(_rec(v=(0, 0, 0.5)), z12, z12, z12, 0.0, 0)
    k, val = gold["vz_half"]
    assert abs(terms[k] - val) < 1e-6
    terms, _ = oracle.reward_terms(_rec(v=(0.5, 0, 0), cmd=(0.0, 0, 0)), z12, z12, z12, 0.0, 0)
    k, val = gold["err_half"]
    assert abs(terms[k] - val) < 1e-6


def test_reward_penalty_terms_closed_form():
    z12 = np.zeros(12, np.float32)
    rng = np.random.default_rng(3)
    rec = _rec(v=(0.2, 0.1, -0.3), w=(0.4, -0.5, 0.1), cmd=(0.5, 0.2, -0.4))
    rec["qd"] = rng.uniform(-2, 2, 12)
    rec["aprev"] = rng.uniform(-1, 1, 12)
    a = rng.uniform(-1, 1, 12).astype(np.float32)
    tau = rng.uniform(-80, 80, 12).astype(np.float32)
    qdd = rng.uniform(-50, 50, 12).astype(np.float32)
    terms, tot = oracle.reward_terms(rec, a, tau, qdd, 0.37, 2)
    dt = 0.02
    qd = rec["qd"].astype(np.float64)
    assert abs(terms[2] - (-4 * dt * 0.09)) < 1e-6
    assert abs(terms[3] - (-0.05 * dt * (0.16 + 0.25))) < 1e-6
    assert abs(terms[4] - (-0.001 * dt * (np.sum(qdd.astype(np.float64) ** 2) + np.sum(qd ** 2)))) < 1e-6
    assert abs(terms[5] - (-0.00002 * dt * np.sum(tau.astype(np.float64) ** 2))) < 1e-6
    rate = (0.5 * (a.astype(np.float64) - rec["aprev"])) / dt
    assert abs(terms[6] - (-0.25 * dt * np.sum(rate ** 2))) < 1e-5
    assert abs(terms[7] - (-0.001 * dt * 2)) < 1e-9
    assert abs(terms[8] - 2 * dt * 0.37) < 1e-7
    assert 0 < terms[0] <= 0.02 and 0 < terms[1] <= 0.01        # φ bounds
    assert np.all(terms[2:8] <= 0)
    assert abs(tot - np.sum(terms.astype(np.float64))) < 1e-6


# ---------------------------------------------------------------- observation
def test_observation_examples():
    env = _env(n=3, flags=0)
    env.reset()
    for i in range(3):
        _place(env, i, 0.5)
    obs = env.observe()
    assert np.all(obs[:, 6:9] == np.array([0, 0, -1], np.float32))  # level pose -> gravity (0,0,-1)
    assert np.all(obs[:, 48:] == np.float32(0.5))                    # flat ground, base 0.5 m
    assert obs.shape[1] == 235
    noisy = oracle.Env(3, env.hf, 1, 1, seed=123, flags=oracle.F_NOISE)
    noisy.state[:] = env.state
    o2 = noisy.observe()
    assert np.all(o2[:, 9:12] == obs[:, 9:12])                      # command noise exactly 0
    assert np.all(o2[:, 36:48] == obs[:, 36:48])                    # no noise on previous actions
    d = (o2 - obs).astype(np.float64)
    assert np.all(np.abs(d[:, 24:36]) <= 1.5) and np.any(d[:, 24:36] != 0)
    assert np.all(np.abs(d[:, 48:]) <= 0.1 + 1e-6)


# ---------------------------------------------------------------- reset / spawn
def test_reset_ranges_and_assignment():
    hf = synth.make_world(10, 20, seed=0, rough=False)
    env = oracle.Env(4096, hf, 10, 20, seed=7)
    env.reset()
    st = env.state
    assert np.all((st["mu"] >= 0.5) & (st["mu"] <= 1.25))
    assert np.all(np.abs(st["cmd"]) <= 1.0)
    assert np.all(st["level"] == 0) and np.all(st["ep_step"] == 0)
    assert np.array_equal(st["col"], np.arange(4096) % 20)
    occ = np.bincount(st["col"] % 5, minlength=5)
    assert set(occ.tolist()) <= {819, 820}
    x, y = st["p"][:, 0], st["p"][:, 1]
    assert np.all(np.abs(x - 4.0) <= 1.0) and np.all(np.abs(y - (8.0 * st["col"] + 4.0)) <= 1.0)
    qn = np.sum(st["quat"].astype(np.float64) ** 2, axis=1)
    assert np.max(np.abs(qn - 1.0)) < 1e-6
    assert np.all(np.abs(st["q"] - QDEF) <= 0.05 + 1e-6)


# ---------------------------------------------------------------- curriculum
def test_curriculum_examples():
    for r in _rows("curriculum_examples.txt"):
        lv, cr, dx, dy, c0, c1, ep, exp = r
        got = oracle.curriculum_level(int(lv), 10, int(cr), float(dx), float(dy), float(c0), float(c1), int(ep), 0)
        assert got == int(exp)
    # loop-back from the top level: uniform in [0, L-1] by multiply-shift
    for w in (0, 0xFFFFFFFF, 0x80000000, 12345678):
        assert oracle.curriculum_level(9, 10, 1, 0, 0, 0, 0, 10, w) == (w * 10) >> 32


def test_curriculum_exhaustive_L3():
    """all 3^6 outcome sequences (cross / under-travel / neither) vs a hand-written machine."""
    import itertools
    for seq in itertools.product(range(3), repeat=6):
        lv_o = lv_h = 0
        for k, ev in enumerate(seq):
            word = (k * 0x9E3779B9) & 0xFFFFFFFF
            crossed = 1 if ev == 0 else 0
            dx = 0.0 if ev == 1 else 100.0
            lv_o = oracle.curriculum_level(lv_o, 3, crossed, dx, 0.0, 1.0, 0.0, 500, word)
            if ev == 0:
                lv_h = lv_h + 1 if lv_h < 2 else (word * 3) >> 32
            elif ev == 1:
                lv_h = max(0, lv_h - 1)
            assert lv_o == lv_h and 0 <= lv_o <= 2


# ---------------------------------------------------------------- env step invariants
def test_env_step_determinism_and_batch_independence():
    hf = synth.make_world(10, 20, seed=0)
    flags = oracle.F_CURRICULUM | oracle.F_NOISE | oracle.F_PUSH | oracle.F_BOOTSTRAP
    e1 = oracle.Env(8, hf, 10, 20, seed=5, flags=flags)
    e2 = oracle.Env(8, hf, 10, 20, seed=5, flags=flags)
    o1, o2 = e1.reset(), e2.reset()
    assert np.array_equal(o1, o2)
    rng = np.random.default_rng(0)
    for _ in range(30):
        a = rng.standard_normal((8, 12)).astype(np.float32)
        r1 = e1.step(a)
        r2 = e2.step(a)
        for x, y in zip(r1, r2):
            assert np.array_equal(x, y)
    assert e1.state.tobytes() == e2.state.tobytes()
    # batch of 8 on rank 0 == envs 4..7 run as "rank 1" of a 4-env world (keyed by global id)
    e3 = oracle.Env(4, hf, 10, 20, seed=5, flags=flags, rank=1)
    e4 = oracle.Env(8, hf, 10, 20, seed=5, flags=flags)
    e3.reset()
    e4.reset()
    assert e3.state.tobytes() == e4.state[4:].tobytes()
    for _ in range(10):
        a = rng.standard_normal((8, 12)).astype(np.float32)
        e3.step(a[4:])
        e4.step(a)
    assert e3.state.tobytes() == e4.state[4:].tobytes()


def test_env_step_flags_timeout_and_reset():
    env = _env(n=4, flags=oracle.F_BOOTSTRAP)
    env.reset()
    for i in range(4):
        _place(env, i, 0.53)
    env.state["ep_step"][0] = 999
    obs, rew, term, to, terms, tobs = env.step(np.zeros((4, 12), np.float32))
    assert to[0] == 1 and term[0] == 0 and env.state["ep_step"][0] == 0   # reset after time-out
    assert np.any(tobs[0] != 0)                                           # terminal obs present
    assert np.all(env.state["ep_step"][1:] == 1)
    # crash: base below r_b -> terminated, reset
    _place(env, 1, 0.1)
    obs, rew, term, to, terms, tobs = env.step(np.zeros((4, 12), np.float32))
    assert term[1] == 1 and to[1] == 0
    # reward breakdown sums to total
    assert np.max(np.abs(terms.sum(1) - rew)) < 1e-6


def test_push_every_500_steps():
    env = _env(n=1, flags=oracle.F_PUSH)
    env.reset()
    _place(env, 0, 50.0)
    env.state["push_timer"][0] = 499
    env.step(np.zeros((1, 12), np.float32))
    assert env.state["push_timer"][0] == 500
    v_before = env.state["v"][0].copy()
    env.step(np.zeros((1, 12), np.float32))
    dv = env.state["v"][0][:2] - v_before[:2]
    assert env.state["push_timer"][0] == 1
    assert np.all(np.abs(dv) <= 1.0) and np.any(dv != 0)


def test_gaussian_noise_moments_and_logp_constant():
    env = _env(n=20000)
    eps = env.action_eps(s=1).astype(np.float64)
    assert abs(eps.mean()) < 0.01 and abs(eps.std() - 1.0) < 0.01
    assert abs(np.mean(eps ** 4) - 3.0) < 0.05
    from oracle import learn
    lp = learn.logp_gauss(np.zeros((1, 12)), np.zeros((1, 12)), np.zeros(12))
    assert abs(lp[0] - (-11.027262398)) < 1e-8


# ---------------------------------------------------------------- shuffle
@pytest.mark.parametrize("B", [1, 2, 3, 1536, 4096, 98304, 100000])
def test_feistel_is_bijection(B):
    keys = oracle.shuffle_keys(42, 0, 3, 5, 1)
    p = oracle.feistel_perm(B, keys)
    assert np.array_equal(np.sort(p), np.arange(B, dtype=np.uint32))
    if B > 1000:
        assert np.mean(p[:-1] < p[1:]) < 0.6                     # actually shuffled


def test_pd_joint_through_the_transition_kp80():
    """PD law through the oracle's transition (DESIGN §3.5 with R24's Kp = 80): a robot in the air (no
    contact, so the joint is decoupled from the base) gets q* - q = 0.1 on one joint.  Four semi-implicit Euler
    substeps of the scalar joint model J q̈ = Kp(q* - q) - Kd q̇ - c_j q̇ (J = 0.25, Kd = 2, c_j = 0.5, dt = 5 ms),
    evaluated here in fp64, fix the last substep's τ and q̈ the transition reports and the joint state it leaves.
    The first substep's torque is Kp·0.1 = 8 N·m; Kp = 50 would give 5 and a different trajectory."""
    env = _env()
    env.reset()
    for j, qs in ((1, 0.1), (8, -0.1), (3, 0.1)):
        _place(env, 0, 5.0)
        a = np.zeros(12, np.float32)
        a[j] = np.float32(2.0 * qs)                       # q* = q_def + 0.5 a  ->  q* - q = qs
        q, qd, taus = 0.0, 0.0, []
        for _ in range(4):
            tau = max(-80.0, min(80.0, 80.0 * (qs - q) - 2.0 * qd))
            taus.append(tau)
            qdd = (tau - 0.5 * qd) / 0.25
            qd += 0.005 * qdd
            q += 0.005 * qd
        assert abs(taus[0] - 80.0 * qs) < 1e-12           # 8 N·m in the first substep
        tau_o, qdd_o, *_ = env.transition_single(0, a)
        assert abs(tau_o[j] - taus[-1]) < 2e-4, (tau_o[j], taus[-1])
        assert abs(qdd_o[j] - qdd) < 1e-3
        assert abs((env.state["q"][0][j] - QDEF[j]) - q) < 1e-6
        assert abs(env.state["qd"][0][j] - qd) < 1e-5
        others = [k for k in range(12) if k != j]
        assert np.all(tau_o[others] == 0.0) and np.all(qdd_o[others] == 0.0)


def test_flight_trajectory_closed_forms():
    """The multi-step transition over 20 policy steps = 80 semi-implicit Euler substeps of a robot
    in flight (no contact), against the closed forms of that integrator, evaluated in fp64 here:
    base free fall v_z(n) = -g dt n, p_z(n) = p_z(0) - g dt² n(n+1)/2 (velocity first, then position with the new
    velocity); torque-free spin about the principal z axis (ω × Iω = 0, so ω stays exactly constant) with the
    first-order quaternion step q + (dt/2) q⊗ω followed by normalisation, which turns the heading by exactly
    2 atan(ω dt / 2) per substep; and one PD-driven joint following the scalar recurrence of S:181 (R24's Kp = 80)
    while the others stay at q* -- the joints are decoupled from the base without contact forces."""
    env = _env()
    env.reset()
    _place(env, 0, 5.0)
    w, th0, dt, g = 2.0, 0.3, 0.005, 9.81
    env.state["w"][0] = (0.0, 0.0, w)
    env.state["quat"][0] = (math.cos(th0 / 2), 0.0, 0.0, math.sin(th0 / 2))
    j, qs = 1, 0.1
    a = np.zeros(12, np.float32)
    a[j] = np.float32(2.0 * qs)
    q, qd = 0.0, 0.0
    for step in range(1, 21):
        tau_o, qdd_o, _, crash, nc, fz = env.transition_single(0, a)
        assert crash == 0 and fz == 0.0
        for _ in range(4):
            tau = max(-80.0, min(80.0, 80.0 * (qs - q) - 2.0 * qd))
            qd += dt * ((tau - 0.5 * qd) / 0.25)
            q += dt * qd
        n = 4 * step
        st = env.state[0]
        assert abs(st["v"][2] - (-g * dt * n)) < 2e-5
        assert abs(st["p"][2] - (5.0 - g * dt * dt * n * (n + 1) / 2)) < 2e-5
        assert st["p"][0] == 4.0 and st["p"][1] == 4.0 and st["v"][0] == 0.0 and st["v"][1] == 0.0
        assert tuple(st["w"]) == (0.0, 0.0, np.float32(w))
        th = th0 + 2.0 * n * math.atan(w * dt / 2.0)
        qt = st["quat"].astype(np.float64)
        assert qt[1] == 0.0 and qt[2] == 0.0
        assert abs(qt[0] - math.cos(th / 2)) < 1e-6 and abs(qt[3] - math.sin(th / 2)) < 1e-6
        assert abs((st["q"][j] - QDEF[j]) - q) < 1e-6 and abs(st["qd"][j] - qd) < 1e-5
        others = [k for k in range(12) if k != j]
        assert np.all(st["q"][others] == QDEF[others]) and np.all(st["qd"][others] == 0.0)


def _ramp_world(a, b, levels=2, cols=2):
    """Heightfield of a plane: node (i, j) -- at the cell centre ((i+1/2)·0.1, (j+1/2)·0.1) -- holds a·i + b·j."""
    i = np.arange(80 * levels, dtype=np.float64)[:, None]
    j = np.arange(80 * cols, dtype=np.float64)[None, :]
    return (a * i + b * j).astype(np.float32)


def _yaw_pitch_quat(yaw, pitch=0.0):
    """(w, x, y, z) of R = R_z(yaw) R_y(pitch)."""
    cy, sy, cp, sp = math.cos(yaw / 2), math.sin(yaw / 2), math.cos(pitch / 2), math.sin(pitch / 2)
    return np.array([cy * cp, -sy * sp, cy * sp, sy * cp])


def _rotmat(q):
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


@pytest.mark.parametrize("yaw", [0.0, math.pi / 2, 0.7])
def test_height_scan_on_a_ramp_rotates_with_heading(yaw):
    """R1-R3: bilinear interpolation is exact on a plane, so on the ramp world
    h(x, y) = a·(10x - 1/2) + b·(10y - 1/2) and scan point k = 11·ix + iy at offset ((ix-8)·0.1, (iy-5)·0.1)
    rotated by the heading ψ must read p_z - h(p + R_z(ψ)·offset).  a != b, so a transposed layout, a wrong
    rotation sense or a swapped axis fails at yaw π/2 and 0.7."""
    a, b = 0.013, 0.029
    hf = _ramp_world(a, b)
    env = oracle.Env(1, hf, 2, 2, seed=1, scan=(17, 11), flags=0)
    env.reset()
    px, py, pz = 8.05, 7.9, 5.0
    env.state["p"][0] = (px, py, pz)
    env.state["quat"][0] = _yaw_pitch_quat(yaw)
    obs = env.observe()[0]
    c, s = math.cos(yaw), math.sin(yaw)
    want = np.zeros(187)
    for ix in range(17):
        for iy in range(11):
            dx, dy = (ix - 8) * 0.1, (iy - 5) * 0.1
            x, y = px + c * dx - s * dy, py + s * dx + c * dy
            want[11 * ix + iy] = pz - (a * (10 * x - 0.5) + b * (10 * y - 0.5))
    got = obs[48:].astype(np.float64)
    assert np.max(np.abs(got - want)) < 2e-5, np.max(np.abs(got - want))
    # and the layout really matters here: the transposed reading (k = 17·iy + ix) is far off
    assert np.max(np.abs(got.reshape(17, 11).T.reshape(-1)[:187] - want)) > 1e-2


def test_reward_heading_frame_at_yaw_pi_over_2():
    """R6 ('the z axis is aligned with gravity'): the tracking terms use the velocity in the heading frame.
    A robot yawed by π/2 moving along world +y at 0.7 m/s, commanded (0.7, 0) in its own frame, tracks perfectly:
    r1 = 1·dt·φ(0) = 0.02, r2 = 0.5·dt = 0.01 (Table 2).  With the frame rotated the wrong way, or not at all,
    the error would be √2·0.7 or 0.7·|(1, -1)| and r1 < 0.0004."""
    z12 = np.zeros(12, np.float32)
    rec = _rec(v=(0.0, 0.7, 0.0), w=(0.0, 0.0, 0.0), cmd=(0.7, 0.0, 0.0))
    rec["quat"] = _yaw_pitch_quat(math.pi / 2)
    terms, _ = oracle.reward_terms(rec, z12, z12, z12, 0.0, 0)
    assert abs(terms[0] - 0.02) < 1e-6 and abs(terms[1] - 0.01) < 1e-6
    rec["v"] = (0.7, 0.0, 0.0)                            # moving along world x = sideways for this robot
    terms, _ = oracle.reward_terms(rec, z12, z12, z12, 0.0, 0)
    assert abs(terms[0] - 0.02 * math.exp(-(0.49 + 0.49) / 0.25)) < 1e-6
    # yaw rate: ω_b = (0, 0, 0.4) at yaw π/2 -> heading-frame ω_z = 0.4 (z is shared), command 0.4 -> r2 = 0.01
    rec["v"] = (0.0, 0.7, 0.0)
    rec["w"] = (0.0, 0.0, 0.4)
    rec["cmd"] = (0.7, 0.0, 0.4)
    terms, _ = oracle.reward_terms(rec, z12, z12, z12, 0.0, 0)
    assert abs(terms[1] - 0.01) < 1e-6


@pytest.mark.parametrize("yaw,pitch", [(0.9, 0.3), (-2.2, -0.45), (math.pi / 2, 0.2)])
def test_observation_body_frame_at_pitched_yawed_pose(yaw, pitch):
    """S:247 / SURVEY O-O: obs[0:3] = Rᵀ v (base-frame linear velocity), obs[3:6] = ω_b, obs[6:9] = Rᵀ (0, 0, -1)
    (projected gravity), with R from the base quaternion -- checked against a numpy rotation at a pitched and
    yawed pose (a transposed R, a wrong quaternion convention or world-frame values fail)."""
    env = _env(flags=0)
    env.reset()
    _place(env, 0, 3.0)
    q = _yaw_pitch_quat(yaw, pitch)
    env.state["quat"][0] = q
    v = np.array([0.6, -0.3, 0.25])
    w = np.array([0.2, 0.5, -0.7])
    env.state["v"][0] = v
    env.state["w"][0] = w
    obs = env.observe()[0].astype(np.float64)
    R = _rotmat(q.astype(np.float32).astype(np.float64))
    assert np.max(np.abs(obs[0:3] - R.T @ v)) < 2e-6
    assert np.max(np.abs(obs[3:6] - w)) < 1e-7
    assert np.max(np.abs(obs[6:9] - R.T @ np.array([0.0, 0.0, -1.0]))) < 2e-6
    # sanity of the fixture itself: pitch tilts gravity into the body x axis
    assert abs(obs[6] - math.sin(pitch)) < 1e-5
