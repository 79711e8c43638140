"""Per-kernel-family achieved HBM GB/s of one H1 solve: SURVEY 8(d) algorithmic
bytes per family (from the hierarchy sizes in a bench line's `details`) over
the kernel time of an ncu launch list summary (cold cache, serialised).

  python tools/kernel_gbs.py profiles/r02e_c3_launches_summary.txt profiles/r02f_c3_bench.json
"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUMMARY, BENCH = sys.argv[1], sys.argv[2]
bench = json.loads(open(BENCH).read().strip().splitlines()[-1])
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6538.9
det = bench["details"]
n, nnzA, nnzP, nit = det["levels"], det["nnz_levels"], det["nnz_P"], det["nit"]
L = len(n) - 1


def ab(nnz, rows):
    return 12 * nnz + 4 * (rows + 1)


def ld(k):  # entries of L + D (forward sweep from zero)
    return (nnzA[k] - n[k]) // 2 + n[k]


B = {  # bytes per PCG iteration
    "fine sweeps (gs_lean, level 0)": 12 * ld(0) + 4 * (n[0] + 1) + 24 * n[0] + ab(nnzA[0], n[0]) + 32 * n[0],
    "coarse sweeps (cluster / grid / row / stream)": sum(12 * ld(k) + 4 * (n[k] + 1) + 24 * n[k] + ab(nnzA[k], n[k])
                                                    + 32 * n[k] for k in range(1, L)),
    "residual SpMV": sum(ab(nnzA[k], n[k]) + 24 * n[k] for k in range(L)),
    "restriction SpMV": sum(ab(nnzP[k], n[k + 1]) + 8 * n[k] + 8 * n[k + 1] for k in range(L)),
    "prolongation SpMV": sum(ab(nnzP[k], n[k]) + 8 * n[k + 1] + 16 * n[k] for k in range(L)),
    "PCG A p (spmv_dot)": ab(nnzA[0], n[0]) + 24 * n[0],
    "coarsest GEMV": 8 * n[L] ** 2 + 16 * n[L],
    "PCG vector updates and dots": (32 + 16 + 24) * n[0],
}
fam = {
    "fine sweeps (gs_lean, level 0)": ("gs_lean_kernel",),
    "coarse sweeps (cluster / grid / row / stream)": ("gs_cluster_kernel", "gs_row_kernel", "gs_stream_kernel",
                                                 "gs_level_kernel", "gs_prepare"),
    "residual SpMV": ("spmv_stream_kernel<1>", "spmv_warp_kernel<1>", "spmv_kernel<1>"),
    "restriction SpMV": ("spmv_stream_kernel<0>", "spmv_warp_kernel<0>", "spmv_kernel<0>"),
    "prolongation SpMV": ("spmv_stream_kernel<2>", "spmv_warp_kernel<2>", "spmv_kernel<2>"),
    "PCG A p (spmv_dot)": ("spmv_dot_kernel",),
    "coarsest GEMV": ("gemv_kernel",),
    "PCG vector updates and dots": ("pcg_xr_kernel", "dot2_kernel", "pcg_p_kernel"),
}
T = {}
its = 0
for line in open(SUMMARY).read().splitlines():
    m = re.match(r"\s*([\d.]+)%\s+(\d+)\s+([\d.]+)\s+(\S.*)$", line)
    if m:
        T[m.group(4).strip()] = int(m.group(2)) * float(m.group(3)) * 1e-6
        if m.group(4).strip().startswith("spmv_dot_kernel"):
            its = int(m.group(2))  # one A p per PCG iteration: the iterations the launch list covers
scale = nit / its if its else 1.0  # kernel time per solve of nit iterations
T = {k: v * scale for k, v in T.items()}
used = set()
print(f"# {os.path.basename(BENCH)}: {nit} PCG iterations, levels {n}; peak {peak:.0f} GB/s (MEASURED_PEAKS.json)")
print(f"# time: {os.path.relpath(SUMMARY, ROOT)} (ncu launch list, cold cache, serialised; {its} iterations listed,")
print(f"# scaled to one solve of {nit}); the prepare kernels")
print("# (rhs permutation / fold / sentinel fill) are counted with the coarse sweeps; bytes: SURVEY 8(d) model")
print(f"{'kernel family':42s} {'MB/iter':>9} {'ms/solve':>9} {'GB/s':>8} {'% peak':>7}")
tb = tt = 0.0
for k in B:
    t = sum(v for name, v in T.items() if any(name.startswith(pfx) for pfx in fam[k]))
    used |= {name for name in T if any(name.startswith(pfx) for pfx in fam[k])}
    bb = B[k] * nit
    tb, tt = tb + bb, tt + t
    print(f"{k:42s} {B[k] / 1e6:9.2f} {t * 1e3:9.2f} {bb / max(t, 1e-12) / 1e9:8.1f} "
          f"{100 * bb / max(t, 1e-12) / 1e9 / peak:6.2f}%")
print(f"{'all':42s} {tb / nit / 1e6:9.2f} {tt * 1e3:9.2f} {tb / tt / 1e9:8.1f} {100 * tb / tt / 1e9 / peak:6.2f}%")
rest = sorted(set(T) - used)
if rest:
    print("# not in a family:", ", ".join(rest))
