"""Multi-rank semantics of the data-parallel path on CPU with the gloo
backend, world_size 2: envs keyed by global id, advantage statistics over the union batch, and the
per-minibatch gradient average over ranks == the gradient of the union minibatch (equal sizes), so the
Adam replicas stay bitwise identical.  Also runs bench.py's reference arm under torchrun."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    import oracle
    from oracle import learn
    import synth
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, T, D, hid = 16, 6, 48, (32, 32, 32)
    hf = synth.make_world(1, 1, rough=False)
    env = oracle.Env(N, hf, 1, 1, seed=9, rank=rank, scan=(0, 0), flags=oracle.F_NOISE | oracle.F_PUSH)
    env.reset()
    rng = np.random.default_rng(100 + rank)  # teacher actions (per-rank streams, seeded)
    obs, rew, term, to = [], [], [], []
    for t in range(T):
        a = rng.standard_normal((N, 12)).astype(np.float32)
        o, r, te, tmo, _, _ = env.step(a)
        obs.append(o); rew.append(r); term.append(te); to.append(tmo)
    st = env.state.copy()
    # union-batch advantage normalisation: global mean/std from all-reduced (count, sum, sum of squares)
    A = np.random.default_rng(7 + rank).standard_normal((T, N))
    stats = torch.tensor([A.size, A.sum(), (A ** 2).sum()], dtype=torch.float64)
    dist.all_reduce(stats)
    n, s1, s2 = stats.tolist()
    mean = s1 / n
    std = np.sqrt((s2 - n * mean * mean) / (n - 1))
    An = (A - mean) / (std + 1e-8)
    # per-rank minibatch gradient, averaged over ranks (the NCCL allreduce of the GPU path)
    theta = synth.init_params(D, hid, seed=3).astype(np.float64)
    p = learn.unpack(theta, D, hid)
    M = 24
    bt = synth.synthetic_storage(1, M, D, seed=50 + rank)
    g, stt = learn.ppo_minibatch(p, bt["obs"][0].astype(np.float64), bt["act"][0].astype(np.float64),
                                 bt["logp"][0].astype(np.float64), bt["V"][0].astype(np.float64),
                                 An.reshape(-1)[:M], bt["r"][0].astype(np.float64), bt["mu"][0].astype(np.float64),
                                 np.zeros(12))
    gt = torch.from_numpy(learn.pack(g, D, hid))
    dist.all_reduce(gt)
    gavg = gt.numpy() / world
    kl = torch.tensor([stt["kl"]], dtype=torch.float64)
    dist.all_reduce(kl)
    th2, *_ = learn.adam_step(theta, gavg, np.zeros_like(theta), np.zeros_like(theta), 0, 1e-3)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), state=st.view(np.uint8), An=An, gavg=gavg, th2=th2,
             kl=kl.numpy() / world)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_semantics(tmp_path):
    import oracle
    from oracle import learn
    import synth
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0, r1 = (np.load(tmp_path / f"rank{r}.npz") for r in (0, 1))
    # (i) env slices keyed by global id == one process over 2N envs
    N, T, D, hid = 16, 6, 48, (32, 32, 32)
    hf = synth.make_world(1, 1, rough=False)
    env = oracle.Env(2 * N, hf, 1, 1, seed=9, scan=(0, 0), flags=oracle.F_NOISE | oracle.F_PUSH)
    env.reset()
    acts = [np.random.default_rng(100 + r) for r in (0, 1)]
    for t in range(T):
        a = np.concatenate([acts[0].standard_normal((N, 12)), acts[1].standard_normal((N, 12))]).astype(np.float32)
        env.step(a)
    whole = env.state.view(np.uint8).reshape(2 * N, -1)
    assert np.array_equal(r0["state"].reshape(N, -1), whole[:N])
    assert np.array_equal(r1["state"].reshape(N, -1), whole[N:])
    # (ii) union normalisation == single-process normalisation of the concatenated batch
    A = np.concatenate([np.random.default_rng(7 + r).standard_normal((T, N)) for r in (0, 1)], axis=1)
    An = learn.normalize_adv(A)
    assert np.allclose(np.concatenate([r0["An"], r1["An"]], axis=1), An, atol=1e-12)
    # (iii) rank-average gradient == gradient of the union minibatch; replicas identical after Adam
    theta = synth.init_params(D, hid, seed=3).astype(np.float64)
    p = learn.unpack(theta, D, hid)
    bts = [synth.synthetic_storage(1, 24, D, seed=50 + r) for r in (0, 1)]
    cat = lambda k: np.concatenate([b[k][0] for b in bts]).astype(np.float64)  # noqa: E731
    adv = np.concatenate([r0["An"].reshape(-1)[:24], r1["An"].reshape(-1)[:24]])
    g, st = learn.ppo_minibatch(p, cat("obs"), cat("act"), cat("logp"), cat("V"), adv, cat("r"), cat("mu"), np.zeros(12))
    # the union loss is the mean over 2M rows; the rank losses are means over M rows -> average of ranks
    assert np.allclose(r0["gavg"], learn.pack(g, D, hid), rtol=1e-10, atol=1e-14)
    assert np.array_equal(r0["gavg"], r1["gavg"]) and np.array_equal(r0["th2"], r1["th2"])
    assert abs(float(r0["kl"][0]) - st["kl"]) < 1e-12


def test_bench_reference_arm_under_torchrun():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus",
           "2", "--steps", "1", "--warmup", "0", "--workload", "c1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    import json
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def _lib_worker(rank, world, port, out_dir):
    """One rank of the product's multi-process setup on CPU: the library is loaded, rank 0 draws the NCCL
    unique id through lg_nccl_unique_id and the process group (gloo here, as torch.distributed carries it on a
    GPU box) delivers it to every rank; each rank validates its own (rank, world) config through the C ABI."""
    sys.path.insert(0, ROOT)
    from paper_2109_11978_b200 import lg
    from paper_2109_11978_b200.context import Config
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        st, raw = lg.lg_nccl_unique_id()
        assert st == 0
        uid = torch.frombuffer(bytearray(raw), dtype=torch.uint8).clone()
    dist.broadcast(uid, 0)
    st, sizes = lg.lg_required_sizes(Config.make(n_envs=64, n_steps=4, rank=rank, world_size=world).to_c())
    bad, _ = lg.lg_required_sizes(Config.make(n_envs=64, n_steps=4, rank=world, world_size=world).to_c())
    np.savez(os.path.join(out_dir, f"lib{rank}.npz"), uid=uid.numpy(), st=st, bad=bad, sizes=np.array(sizes))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_library_setup(tmp_path):
    from paper_2109_11978_b200 import build
    build.build()
    port = _free_port()
    mp.spawn(_lib_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0, r1 = (np.load(tmp_path / f"lib{r}.npz") for r in (0, 1))
    assert np.array_equal(r0["uid"], r1["uid"]) and r0["uid"].any()    # every rank holds rank 0's id
    assert int(r0["st"]) == 0 and int(r1["st"]) == 0                   # LG_OK for rank 0 and rank 1 of 2
    assert int(r0["bad"]) == 2 and int(r1["bad"]) == 2                 # rank >= world: LG_ERR_RANGE
    assert np.array_equal(r0["sizes"], r1["sizes"])                    # identical per-rank layouts
    from paper_2109_11978_b200 import lg
    assert lg._lib.lg_group_create(None, 2, None) == 1                  # LG_ERR_INVALID_ARG
