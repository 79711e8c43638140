set -x
for w in fwd5 fwd3; do
  timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gs_stream -c 1 \
    -o /tmp/r2_$w python tools/profile_solve.py c3 $w > gpurun_out/r2c_ncu_$w.log 2>&1
  ncu -i /tmp/r2_$w.ncu-rep --page details --csv > gpurun_out/r2c_${w}_details.csv 2>&1
  ncu -i /tmp/r2_$w.ncu-rep --page source --csv --print-source sass > gpurun_out/r2c_${w}_sass.csv 2>&1
  ls -la gpurun_out/r2c_${w}_*
done
