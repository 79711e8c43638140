set -x
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -3 | tee gpurun_out/r2p_gpu_tests.log
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r2p_b200_c3.json 2> gpurun_out/r2p_b200_c3.err
python -c "
import json; d=json.loads(open('gpurun_out/r2p_b200_c3.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'cycle', d['cycle'], 'nit', d['details']['nit'], d['details'].get('history_rel_max_vs_oracle'))
print('roofline', d['roofline']); print('h2', d.get('h2',{}).get('value'))
for s in d['sweeps'][:4]: print(s['level'], s['rows'], s['kernel'], s['sweep'][:8], round(s['ms']*1e3,1), 'us', round(s['gbs'],1))
"
tail -3 gpurun_out/r2p_b200_c3.err
