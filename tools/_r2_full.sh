set -x
timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -8
timeout 900 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_b200_c3.json 2> gpurun_out/r2d_b200_c3.err
python -c "
import json; d=json.loads(open('gpurun_out/r2d_b200_c3.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'cycle', d['cycle']['ms'], 'nit', d['details']['nit'], 'h2', d.get('h2',{}).get('value'))
for k in d['sweeps']: print(k['level'], k['kernel'], k['sweep'][:8], round(k['ms']*1e3,1), 'us')
"
