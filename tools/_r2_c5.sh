# C5 (3D jump 320^3) on one B200: fit, coarsest spectrum and pseudo-inverse thresholds, oracle check,
# then the bench line (B200 arm, then the reference arm on the cached hierarchy).
set -x
free -g | head -2
timeout 2400 python tools/c5_pinv.py 1e-14 1e-13 1e-12 1e-11 1e-10 1e-9 1e-8 > gpurun_out/r2_c5_pinv.log 2>&1
tail -20 gpurun_out/r2_c5_pinv.log
timeout 1800 python bench.py --config c5 --steps 5 --warmup 3 --no-h2 > gpurun_out/r2_c5_bench.json 2> gpurun_out/r2_c5_bench.err
tail -c 2500 gpurun_out/r2_c5_bench.json; tail -5 gpurun_out/r2_c5_bench.err
timeout 1800 python bench.py --impl reference --config c5 --steps 2 --warmup 1 > gpurun_out/r2_c5_ref.json 2> gpurun_out/r2_c5_ref.err
cat gpurun_out/r2_c5_ref.json; tail -5 gpurun_out/r2_c5_ref.err
