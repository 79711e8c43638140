# ncu --set full of the C3 sweeps: the fine lean wavefront (fwd, bwd), a row-sweep level, a level-set level.
set -x
for w in fwd0 bwd0 fwd1 bwd1 fwd3 fwd5 bwd5; do
  timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -c 3 \
    -o gpurun_out/r2_c3_$w python tools/profile_solve.py c3 $w > gpurun_out/r2_c3_ncu_$w.log 2>&1
done
ls -la gpurun_out/
