"""Critical-path model of the distributed factorization for
P = 1, 2, 4, 8 at c3 (strong scaling) and the bench's weak-scaling shapes
(n = 10000 P^(1/3)).  Inputs: per-step component times measured on ONE B200
(profiles/r02_timeline.txt: in-situ DGEMM rate, chain and panel-QR latencies)
and ASSUMED NCCL costs on NVSwitch (no multi-GPU box was reachable: latency
alpha per collective, bus bandwidth for large allreduces / broadcasts).
Not a measurement.  usage: python tools/dist_model.py"""
import math

R_GEMM = 32.0e12      # in-situ DGEMM rate per GPU, early c3 steps measured 33 TF (r02 timeline), late ~25-30
CHAINS = 0.85e-3      # per step, redundant on every rank: 2 re-orthonormalisations + QR(Y) (measured, late steps)
PQR = 0.65e-3         # column panel QR on the owner (measured ~0.55-0.75 ms)
TAIL = 6.0e-3         # last SVD chunk + folds after the loop (measured ~6-7 ms at c3)
ALPHA = 25e-6         # NCCL latency per collective (assumed)
BW = 350e9            # NCCL allreduce bus bandwidth on NVSwitch, bytes/s (assumed; NVLS can exceed it)


def allreduce(nbytes, P):
    return 0.0 if P == 1 else ALPHA + 2 * (P - 1) / P * nbytes / BW


def bcast(nbytes, P):
    return 0.0 if P == 1 else ALPHA + nbytes / BW


def model(n, P, b=256, q=2):
    m = n
    t = 0.0
    parts = {"gemm": 0.0, "chains": 0.0, "pqr_exposed": 0.0, "comm": 0.0}
    steps = (n - 1) // b
    for i in range(1, steps + 1):
        r0 = b * (i - 1)
        mi = ni = n - r0
        fl = (2 + 4 * q) * mi * ni * b + 4 * m * ni * b + 4 * mi * (ni - b) * b
        g = fl / P / R_GEMM
        upd = 2 * m * (ni - b) * b / P / R_GEMM
        c = q * allreduce(8 * b * b, P) + q * allreduce(8 * mi * b, P) + allreduce(8 * b * b, P) \
            + allreduce(16 * b * b, P) + allreduce(8 * m * b, P) + bcast(8 * (mi * b + 2 * b * b), P)
        parts["gemm"] += g
        parts["chains"] += CHAINS
        parts["pqr_exposed"] += max(0.0, PQR - upd)
        parts["comm"] += c
    t = sum(parts.values()) + TAIL
    return t, parts


if __name__ == "__main__":
    F = lambda n, q=2: (5 + 2 * q) * n ** 3 - (3 + 2 * q) * n ** 3 / 3  # noqa: E731
    print("| P | workload | model ms | GEMM | chains | panel QR exposed | collectives | tail | TF/GPU | efficiency |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    t1, _ = model(10000, 1)
    for P in (1, 2, 4, 8):
        for kind in ("strong", "weak"):
            if P == 1 and kind == "weak":
                continue
            n = 10000 if kind == "strong" else round(10000 * P ** (1 / 3))
            t, p = model(n, P)
            tf = F(n) / t / P / 1e12
            eff = (t1 / (P * t)) if kind == "strong" else t1 / t
            print(f"| {P} | {kind} n={n} | {1e3 * t:.0f} | {1e3 * p['gemm']:.0f} | {1e3 * p['chains']:.0f} | "
                  f"{1e3 * p['pqr_exposed']:.0f} | {1e3 * p['comm']:.0f} | {1e3 * TAIL:.0f} | {tf:.1f} | {eff:.2f} |")
