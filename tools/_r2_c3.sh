# round 2: C3 bench, both arms back to back (reference first, as the driver runs them), then the
# ncu launch list of one C3 H1 solve.
set -x
nproc; lscpu | grep "Model name"
timeout 1500 python bench.py --impl reference --config c3 --steps 3 --warmup 1 > gpurun_out/r2_ref_c3.json 2> gpurun_out/r2_ref_c3.err
timeout 900 python bench.py --config c3 --steps 10 --warmup 3 > gpurun_out/r2_b200_c3.json 2> gpurun_out/r2_b200_c3.err
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c3_launches.csv python tools/profile_solve.py c3 solve > gpurun_out/r2_c3_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_c3_launches.csv > gpurun_out/r2_c3_launches_summary.txt
tail -c 3000 gpurun_out/r2_ref_c3.json; tail -c 6000 gpurun_out/r2_b200_c3.json; head -40 gpurun_out/r2_c3_launches_summary.txt
