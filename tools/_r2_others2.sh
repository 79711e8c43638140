# C2 and C4 bench lines with the cluster / grid sweeps (GPU fit, untimed)
set -x
for c in c2 c4; do
  timeout 1800 python bench.py --config $c --steps 5 --warmup 3 --no-h2 > gpurun_out/r2o_${c}_bench.json 2> gpurun_out/r2o_${c}_bench.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2o_${c}_bench.json').read().strip().splitlines()[-1])
print('$c value', d['value'], 'e2e', d['e2e']['value'], 'cycle', d['cycle']['ms'], 'nit', d['details']['nit'], d['details'].get('oracle_nit'), d['details'].get('history_rel_max_vs_oracle'), 'cpu', d.get('cpu_baseline',{}).get('value'))
for s in d['sweeps']: print(s['level'], s['rows'], s['kernel'], s['sweep'][:8], round(s['ms']*1e3,1), 'us')
"
done
