"""DESIGN R28, pinned on the oracle (CPU): how far one PPO update (5 x 4 minibatches, Alg. 1 + Adam) moves when
the MLP's GEMM operands are rounded at the GPU path's rounding points, against the exact fp64 update.

Adam divides each moment by its own scale, so a gradient element whose sign is decided by less than the
operand rounding error flips a whole ±α step: the parameter drift of a complete update is governed by the
*format* of the operands, not by the bf16 gradient tolerance (2e-2) of north_star.  Measured here on an
oracle rollout (C3 network, 256 envs x 24 steps): fp32 operands stay far inside the north_star drift bound
of 1e-3, bf16 operands -- the format north_star prescribes for the MLP -- cannot meet it against the exact
update even in the oracle itself, at every rounding point alone.  Hence R28: the 1e-3 bound is applied
against the oracle evaluated at the GPU's bf16 rounding points, and the drift against the exact oracle is
bounded by the oracle's own bf16-vs-fp64 gap + 1e-3."""
import numpy as np
import pytest

import oracle
from oracle import learn
import synth


@pytest.fixture(scope="module")
def batch():
    N, T, D, hid = 256, 24, 235, (512, 256, 128)
    hf = synth.make_world(4, 5, seed=3, rough=True)
    theta = synth.init_params(D, hid, seed=11).astype(np.float64)
    env = oracle.Env(N, hf, 4, 5, seed=11)
    obs = env.reset()
    p = learn.unpack(theta, D, hid)
    ls = p["logstd"]
    bt = {k: [] for k in ("obs", "act", "mu", "logp", "V", "r", "b", "term", "timeout")}
    for _ in range(T):
        o = learn.round_bf16(obs)                       # the rollout rows are bf16 on the GPU
        mu, _ = learn.mlp_forward(p, o, "a")
        a = mu + np.exp(ls) * env.action_eps()
        v, _ = learn.mlp_forward(p, o, "c")
        obs, r, te, to, _, _ = env.step(a.astype(np.float32))
        for k, x in (("obs", o), ("act", a), ("mu", mu), ("logp", learn.logp_gauss(a, mu, ls)), ("V", v[:, 0]),
                     ("r", r), ("b", np.zeros(N)), ("term", te), ("timeout", to)):
            bt[k].append(x)
    bt = {k: np.stack(v) for k, v in bt.items()}
    bt["V_T"] = learn.mlp_forward(p, learn.round_bf16(obs), "c")[0][:, 0]
    bt["logstd_old"] = ls.copy()
    perms = [oracle.feistel_perm(N * T, oracle.shuffle_keys(11, 0, 0, 5, e)) for e in range(5)]
    return theta, bt, perms, D, hid


def _update(batch, quant):
    theta, bt, perms, D, hid = batch
    z = np.zeros_like(theta)
    th, _, _, t, alpha, st = learn.ppo_update(theta, z, z.copy(), 0, 1e-3, bt, perms, D, hid, quant=quant)
    return th, [x.get("alpha") for x in st]


def test_update_drift_is_set_by_the_operand_format(batch):
    ref, a_ref = _update(batch, None)
    size = np.linalg.norm(ref - batch[0]) / np.linalg.norm(ref)
    rows = {}
    for q in ("fp32", "tf32", "bf16", "bf16@w", "bf16@h", "bf16@dz", "bf16@wb"):
        th, al = _update(batch, q)
        assert al == a_ref, q                            # Alg. 1 takes the same branches: drift is Adam's
        rows[q] = np.linalg.norm(th - ref) / np.linalg.norm(ref)
    print(f"\nupdate size {size:.3e}; drift vs exact fp64 update: " +
          ", ".join(f"{q} {d:.2e}" for q, d in rows.items()))
    assert rows["fp32"] < 1e-5                           # fp32 operands: far inside north_star's 1e-3
    assert rows["bf16"] > 1e-3                           # bf16 operands: outside it, in the oracle itself
    for q in ("bf16@w", "bf16@h", "bf16@dz", "bf16@wb"):
        assert rows[q] > 5e-4, q                         # every single bf16 rounding point contributes
    assert rows["tf32"] < rows["bf16"]
