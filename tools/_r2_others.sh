# current numbers on the other configurations (B200 arm only, short)
set -x
for c in c1 c2 c4; do
  timeout 1800 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2y_b200_$c.json 2> gpurun_out/r2y_b200_$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2y_b200_$c.json').read().strip().splitlines()[-1])
print('$c', 'value', d['value'], 'e2e', d['e2e']['value'], 'cycle', d['cycle']['ms'], 'nit', d['details']['nit'], 'h2', (d.get('h2') or {}).get('value'), (d.get('h2') or {}).get('nit'), 'roof', d['roofline']['kernel'], d['roofline']['frac'])
"
done
