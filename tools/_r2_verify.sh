# round 2: GPU suite, sanitizers, ncu of the C3 roofline kernel, C3 bench + launch list
set -x
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -15 | tee gpurun_out/r2f_gpu_tests.log
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_gs.py > gpurun_out/r2f_sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2f_sanitize_$tool.log
  tail -4 gpurun_out/r2f_sanitize_$tool.log
done
for w in fwd0 bwd0; do
  timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gs_lean -c 1 \
    -o /tmp/r2f_$w python tools/profile_solve.py c3 $w > gpurun_out/r2f_ncu_$w.log 2>&1
  ncu -i /tmp/r2f_$w.ncu-rep --page details --csv > gpurun_out/r2f_c3_${w}_details.csv 2>&1
  ncu -i /tmp/r2f_$w.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/r2f_c3_${w}_raw.csv 2>&1
done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_c3_launches.csv python tools/profile_solve.py c3 solve > gpurun_out/r2f_c3_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r2f_c3_launches.csv > gpurun_out/r2f_c3_launches_summary.txt
head -30 gpurun_out/r2f_c3_launches_summary.txt
