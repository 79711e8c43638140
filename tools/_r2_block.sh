set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "blocked or structures or stream or vcycle" 2>&1 | tail -4
timeout 900 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-h2 > gpurun_out/r2e_b200_c3.json 2> gpurun_out/r2e_b200_c3.err
python -c "
import json; d=json.loads(open('gpurun_out/r2e_b200_c3.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'cycle', d['cycle']['ms'], 'nit', d['details']['nit'])
for k in d['sweeps']: print(k['level'], k['kernel'], k['sweep'][:8], round(k['ms']*1e3,1), 'us')
"
tail -3 gpurun_out/r2e_b200_c3.err
