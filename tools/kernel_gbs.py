"""Per-kernel achieved HBM GB/s of one C2 H1 solve (SURVEY 8(d) byte model)
from the committed ncu launch list summary (cold-cache, serialised launches)
and the fitted hierarchy's sizes in the committed bench line:

  python tools/kernel_gbs.py [launch_summary.txt] [bench_line.json] > profiles/r01c_c2_kernel_gbs.txt
"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUMMARY = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r01b_c2_launches_summary.txt")
BENCH = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", "r01c_bench_c2.json")
bench = json.loads(open(BENCH).read().strip().splitlines()[-1])
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6518.0
n = bench["config"]["levels"]
gal = bench["galerkin"]["levels"]
nnzA = [g["nnz_A"] for g in gal] + [gal[-1]["nnz_Ac"]]
nnzP = [g["nnz_P"] for g in gal]
L = len(n) - 1                       # coarsest = n[L], dense inverse
nit = bench["config"]["nit"]


def ab(nnz, rows):
    return 12 * nnz + 4 * (rows + 1)


# algorithmic bytes per PCG iteration, per kernel family (fine level k = 0, coarse 1..L-1)
B = {
    "gs_lean fwd (level 0, from x=0)": ab(nnzA[0], n[0]) + 24 * n[0],
    "gs_lean bwd (level 0, from x)": ab(nnzA[0], n[0]) + 32 * n[0],
    "coarse sweeps, row + level-set (L1..)": sum(2 * ab(nnzA[k], n[k]) + 56 * n[k] for k in range(1, L)),
    "gs_prepare (all levels, both sweeps)": sum(28 * n[k] * 2 + 6 * nnzA[k] + 8 * n[k] for k in range(L)),
    "spmv<1> residual": sum(ab(nnzA[k], n[k]) + 24 * n[k] for k in range(L)),
    "spmv<0> restriction": sum(ab(nnzP[k], n[k + 1]) + 8 * n[k] + 8 * n[k + 1] for k in range(L)),
    "spmv<2> prolongation": sum(ab(nnzP[k], n[k]) + 8 * n[k + 1] + 16 * n[k] for k in range(L)),
    "spmv_dot (PCG A p)": ab(nnzA[0], n[0]) + 24 * n[0],
    "gemv (coarsest inverse)": 8 * n[L] ** 2 + 16 * n[L],
    "pcg_xr + dot2 + pcg_p": (32 + 16 + 24) * n[0],
}
# kernel time per solve from the launch list summary
summ = open(SUMMARY).read()
T = {}
for line in summ.splitlines():
    m = re.match(r"\s*([\d.]+)%\s+(\d+)\s+([\d.]+)\s+(\S.*)$", line)
    if m:
        T[m.group(4).strip()] = int(m.group(2)) * float(m.group(3)) * 1e-6


def tt(*names):
    return sum(T.get(x, 0.0) for x in names)


lean = sorted(x for x in T if x.startswith("gs_lean_kernel"))
t = {
    "gs_lean fwd (level 0, from x=0)": T[lean[0]],
    "gs_lean bwd (level 0, from x)": T[lean[1]],
    "coarse sweeps, row + level-set (L1..)": tt("gs_row_kernel<0>", "gs_row_kernel<false>",
                                             "gs_level_kernel<0, 1>", "gs_level_kernel<false, 1>",
                                             "gs_level_kernel<0, 2>", "gs_level_kernel<false, 2>"),
    "gs_prepare (all levels, both sweeps)": tt("gs_prepare_kernel", "gs_prepare_fold_warp_kernel"),
    "spmv<1> residual": tt("spmv_kernel<1>", "spmv_warp_kernel<1>"),
    "spmv<0> restriction": tt("spmv_kernel<0>", "spmv_warp_kernel<0>"),
    "spmv<2> prolongation": tt("spmv_kernel<2>", "spmv_warp_kernel<2>"),
    "spmv_dot (PCG A p)": T["spmv_dot_kernel"],
    "gemv (coarsest inverse)": T["gemv_kernel"],
    "pcg_xr + dot2 + pcg_p": tt("pcg_xr_kernel", "dot2_kernel", "pcg_p_kernel"),
}
print(f"# C2 H1 solve, {nit} PCG iterations; levels {n}; peak {peak:.0f} GB/s (MEASURED_PEAKS.json copy)")
print(f"# time: ncu launch list ({os.path.relpath(SUMMARY, ROOT)}, cold cache, serialised);")
print("# bytes: SURVEY 8(d) model per kernel family (A_k: 12 nnz + 4 (n+1); vectors 8 B/entry)")
print(f"{'kernel family':40s} {'MB/iter':>9} {'ms/solve':>9} {'GB/s':>8} {'% peak':>7}")
tot_b = tot_t = 0.0
for k in B:
    bb, tt = B[k] * nit, t[k]
    tot_b += bb
    tot_t += tt
    print(f"{k:40s} {B[k] / 1e6:9.2f} {tt * 1e3:9.2f} {bb / tt / 1e9:8.1f} {100 * bb / tt / 1e9 / peak:6.2f}%")
print(f"{'all':40s} {tot_b / nit / 1e6:9.2f} {tot_t * 1e3:9.2f} {tot_b / tot_t / 1e9:8.1f} "
      f"{100 * tot_b / tot_t / 1e9 / peak:6.2f}%")
