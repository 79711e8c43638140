set -x
timeout 1200 python tools/h1h2_ab.py c3 "" "stream_gs=False" "stream_max_rows=1024" "stream_max_rows=2048" 2>&1 | grep "\["
timeout 2400 python bench.py --config c5 --steps 5 --warmup 3 --no-h2 > gpurun_out/r2h_c5_bench.json 2> gpurun_out/r2h_c5_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2h_c5_bench.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'cycle', d['cycle'], 'nit', d['details']['nit'], d['roofline'])
for k in d['sweeps']: print(k['level'], k['kernel'], k['sweep'][:8], round(k['ms']*1e3,1), 'us', round(k['gbs'],1))
print(d.get('cpu_baseline'), d.get('cpu_baseline_1core'))
"
tail -3 gpurun_out/r2h_c5_bench.err
