set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "stream" 2>&1 | tail -15
timeout 900 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-h2 > gpurun_out/r2b_b200_c3.json 2> gpurun_out/r2b_b200_c3.err
python -c "
import json; d=json.loads(open('gpurun_out/r2b_b200_c3.json').read().strip().splitlines()[-1])
print('value', d['value'], 'cycle', d['cycle'], 'nit', d['details']['nit'])
for k in d['sweeps']: print(k['level'], k['kernel'], k['sweep'][:8], round(k['ms']*1e3,1), 'us', round(k['gbs'],1))
"
tail -5 gpurun_out/r2b_b200_c3.err
