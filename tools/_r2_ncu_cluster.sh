# ncu evidence for the cluster / grid sweeps on C3 (after the plain runs): launch list of the bench command,
# then --set full captures of the grid form (level 1), the cluster form (level 4) and the fine wavefront.
set -x
timeout 1500 python bench.py --steps 2 --warmup 3 --no-h2 --no-cpu-baseline > gpurun_out/r2m_c3_plain.json 2> gpurun_out/r2m_c3_plain.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/r2m_c3_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-h2 --no-cpu-baseline > gpurun_out/r2m_c3_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r2m_c3_launches.csv > gpurun_out/r2m_c3_launches_summary.txt
gzip -f gpurun_out/r2m_c3_launches.csv
for w in fwd1 bwd1 fwd4 bwd0; do
  timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -c 3 \
    -f -o gpurun_out/r2m_c3_$w python tools/profile_solve.py c3 $w > gpurun_out/r2m_c3_ncu_$w.log 2>&1
  ncu -i gpurun_out/r2m_c3_$w.ncu-rep --page details --csv > gpurun_out/r2m_c3_${w}_details.csv 2>/dev/null
  ncu -i gpurun_out/r2m_c3_$w.ncu-rep --page raw --csv > gpurun_out/r2m_c3_${w}_raw.csv 2>/dev/null
  rm -f gpurun_out/r2m_c3_$w.ncu-rep
done
head -30 gpurun_out/r2m_c3_launches_summary.txt
