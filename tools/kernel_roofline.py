"""Per-kernel roofline table from one `ncu --set full` capture of a window of bench.py launches that covers
every kernel type once (rollout step, bootstrap / V(o_T) critic, GAE, one full minibatch).

usage: python tools/kernel_roofline.py REP [ROUND] > profiles/ROUND_roofline.md

Achieved rates use ncu's serialised per-launch duration (clock-control none, caches flushed between
launches, so DRAM bytes are cold-cache figures). GEMM FLOPs are the algorithmic 2*M*N*K of the launch,
identified by its position in the minibatch (gather, L1, L2, L3, loss, reduce, dW3, dX3, dX2, dW2, dW1,
Adam + next gather); the GEMMs before the minibatch are the time-out bootstrap critic (V(o_T) is the fused
policy kernel's critic half). Peaks: MEASURED_PEAKS.json (bf16 sustained, HBM copy)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3}

# C3 shapes (4096 envs x 24 steps, minibatch 24576, D = 235 (Dp 240), MLP 512-256-128, both nets)
MB, N, DP, H0, H1, H2 = 24576, 4096, 240, 512, 256, 128
UPDATE = {  # name in minibatch order -> FLOPs
    "L1": 2 * MB * 2 * H0 * DP, "L2": 2 * 2 * MB * H1 * H0, "L3": 2 * 2 * MB * H2 * H1,
    "dW3": 2 * 2 * H2 * H1 * MB, "dX3": 2 * 2 * MB * H1 * H2, "dW2": 2 * 2 * H1 * H0 * MB,
    "dX2": 2 * 2 * MB * H0 * H1, "dW1": 2 * 2 * H0 * DP * MB,
}
CRITIC = {"cL1": 2 * N * H0 * DP, "cL2": 2 * N * H1 * H0, "cL3": 2 * N * H2 * H1}
POLICY = 2 * 2 * N * (DP * H0 + H0 * H1 + H1 * H2)


def peaks():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        flat = json.dumps(p)
        hbm = bf16 = None
        for k, v in p.items():
            if isinstance(v, (int, float)):
                if "hbm" in k.lower() and hbm is None:
                    hbm = float(v)
                if "bf16" in k.lower() and "sus" in k.lower():
                    bf16 = float(v)
        return hbm or 6468.3, bf16 or 1413.1, "MEASURED_PEAKS.json" if flat else "fallback"
    except OSError:
        return 6468.3, 1413.1, "fallback"


def main(rep, rnd="r01"):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]

    def val(d, u, k):
        v = d.get(k, "")
        if v in ("", "n/a"):
            return 0.0
        return float(v.replace(",", "")) * SCALE.get(u.get(k, ""), 1.0)

    hbm_peak, tc_peak, src = peaks()
    out = []
    seq, crit = [], []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("lg::", "")
        t = val(d, u, "gpu__time_duration.sum")
        dram = val(d, u, "dram__bytes_read.sum") + val(d, u, "dram__bytes_write.sum")
        tens = val(d, u, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")
        l2 = val(d, u, "lts__throughput.avg.pct_of_peak_sustained_elapsed")
        issue = val(d, u, "smsp__issue_active.avg.pct_of_peak_sustained_active")
        out.append(dict(name=name, grid=d["Grid Size"], t=t, dram=dram, tens=tens, l2=l2, issue=issue))
    # label GEMMs by position: the minibatch starts after k_gather
    labels = [""] * len(out)
    for i, e in enumerate(out):
        if e["name"].startswith("k_gather"):
            # launch order of a minibatch: layer 1, layer 2, layer 3 + the PPO loss epilogue (one kernel), the head
            # reduction (side stream), dW3, dX3, dX2, dW2, dW1, then Adam + the next gather
            order = ["L1", "L2", "L3", None, "dW3", "dX3", "dX2", "dW2", "dW1"]
            for k, lab in enumerate(order, start=1):
                if i + k < len(out) and lab:
                    labels[i + k] = lab
            break
    # GEMMs before the minibatch: the time-out bootstrap critic chain (V(o_T) runs in the fused policy kernel)
    first_gather = next((i for i, e in enumerate(out) if e["name"].startswith("k_gather")), len(out))
    for i, e in enumerate(out[:first_gather]):
        if e["name"].startswith("k_gemm_tc") and not labels[i]:
            labels[i] = "boot"
    out, labels = out[:first_gather + 11], labels[:first_gather + 11]  # one minibatch (its Adam + next gather)
    print(f"# {rnd}: per-kernel roofline fractions (`ncu --set full --clock-control none`, one launch of each kernel)\n")
    print(f"Peaks: bf16 dense {tc_peak:.0f} TFLOP/s sustained, HBM {hbm_peak:.0f} GB/s ({src}). Durations are ncu's "
          "serialised, cold-cache launch times (shares agree with the bench's in-graph times; absolutes are higher).\n")
    print("| kernel | role | grid | µs | roofline | achieved | fraction of peak | limiter (counters) | tensor pipe % | DRAM GB/s | L2 % | issue % |")
    print("|---|---|---|---:|---|---:|---:|---|---:|---:|---:|---:|")
    seen = set()
    for e, lab in zip(out, labels):
        key = (e["name"], lab)
        if key in seen:
            continue
        seen.add(key)
        gbs = e["dram"] / e["t"] / 1e9 if e["t"] else 0.0
        if lab in UPDATE or lab in CRITIC or e["name"].startswith("k_policy_fused"):
            fl = UPDATE.get(lab) or CRITIC.get(lab) or POLICY
            ach = fl / e["t"] / 1e12
            bound, achs, frac = "tensor", f"{ach:.0f} TFLOP/s", ach / tc_peak
        else:
            bound, achs, frac = "hbm", f"{gbs:.0f} GB/s", gbs / hbm_peak
        role = {"L1": "forward layer 1 (both nets)", "L2": "forward layer 2", "L3": "forward layer 3 + PPO loss epilogue",
                "dW3": "weight grad layer 3", "dX3": "input grad layer 3", "dW2": "weight grad layer 2",
                "dX2": "input grad layer 2", "dW1": "weight grad layer 1", "cL1": "critic L1 on o_T",
                "cL2": "critic L2 on o_T", "cL3": "critic L3 on o_T",
                "boot": "time-out bootstrap critic (device-sized M; empty here)"}.get(lab, "")
        role = role or {"k_policy_fused": "rollout policy (3 fused layers + heads + sampling)",
                        "k_env_step": "transition, reward, flags, curriculum, reset", "k_env_obs": "observation + height scan + noise",
                        "k_heads": "value scatter (time-out bootstrap)", "k_gae": "GAE reverse scan",
                        "k_perm": "Feistel shuffle (5 epochs)", "k_gather": "minibatch gather", "k_loss_heads": "heads + PPO loss + dZ3",
                        "k_reduce_heads": "head-gradient reduction", "k_adam": "Alg. 1 + Adam + weight shadows",
                        "k_adam_gather": "Alg. 1 + Adam + shadows, with the next minibatch's gather"}.get(e["name"], "")
        dram_pct = gbs / hbm_peak * 100
        if bound == "tensor" and e["tens"] >= 15:
            lim = "tensor / epilogue traffic"
        elif e["issue"] >= 40:
            lim = "instruction issue"
        elif dram_pct >= 25:
            lim = "HBM"
        elif e["t"] < 6e-6:
            lim = "launch (tiny)"
        else:
            lim = "latency"
        print(f"| `{e['name']}` | {role} | {e['grid']} | {e['t'] * 1e6:.1f} | {bound} | {achs} | {frac:.3f} | {lim} | "
              f"{e['tens']:.1f} | {gbs:.0f} | {e['l2']:.1f} | {e['issue']:.1f} |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "r01")
