set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "short_chain or cluster" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_reference_large.py -x -q -m gpu 2>&1 | tail -3
timeout 1800 python bench.py --config c4 --steps 5 --warmup 3 --no-h2 > gpurun_out/r2o_c4_bench.json 2> gpurun_out/r2o_c4_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2o_c4_bench.json').read().strip().splitlines()[-1])
print('c4 value', d['value'], 'e2e', d['e2e']['value'], 'cycle', d['cycle']['ms'], 'nit', d['details']['nit'], d['details'].get('oracle_nit'), d['details'].get('history_rel_max_vs_oracle'), 'cpu', d.get('cpu_baseline',{}).get('value'))
for s in d['sweeps']: print(s['level'], s['rows'], s['kernel'], s['sweep'][:8], round(s['ms']*1e3,1), 'us')
"
tail -3 gpurun_out/r2o_c4_bench.err
