# ncu evidence for this round's kernels (run on the GPU box, one process at a time)
set -x
# launch list of one default bench solve (cold, serialised per-launch times)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/r1b_c2_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-h2 --no-galerkin > gpurun_out/r1b_ncu_launch.log 2>&1
# Galerkin product kernels on C2's fine level (block prolongator of the reference's shape)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spgemm_smem_kernel -c 2 -o gpurun_out/r1b_galerkin_spgemm python tools/galerkin_bench.py --reps 1 > gpurun_out/r1b_ncu_gk.log 2>&1
