# C5 with the cluster sweeps on levels 5-7: bench line (GPU fit, cached under /tmp), then an ncu launch list of the same command
set -x
timeout 3000 python bench.py --config c5 --steps 5 --warmup 3 --no-h2 --no-cpu-baseline > gpurun_out/r2i_c5_bench.json 2> gpurun_out/r2i_c5_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2i_c5_bench.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'cycle', d['cycle'], 'nit', d['details']['nit'], d['roofline'])
for k in d['sweeps']: print(k['level'], k['kernel'], k['sweep'][:8], round(k['ms']*1e3,1), 'us', round(k['gbs'],1))
"
tail -3 gpurun_out/r2i_c5_bench.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r2i_c5_launches.csv python bench.py --config c5 --steps 1 --warmup 3 --no-h2 --no-cpu-baseline > gpurun_out/r2i_c5_ncu.log 2>&1
tail -2 gpurun_out/r2i_c5_ncu.log
gzip -f gpurun_out/r2i_c5_launches.csv
