# final round-2 evidence, the driver's order: reference arm first (CPU-only setup, writes the hierarchy cache), then the
# B200 arm, GPU suite, smoke
set -x
rm -rf /tmp/mvamg_hcache
timeout 2400 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2z_ref_c3.json 2> gpurun_out/r2z_ref_c3.err
tail -c 600 gpurun_out/r2z_ref_c3.json
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r2z_b200_c3.json 2> gpurun_out/r2z_b200_c3.err
python -c "
import json; d=json.loads(open('gpurun_out/r2z_b200_c3.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'cycle', d['cycle'], 'nit', d['details']['nit'], d['details'].get('history_rel_max_vs_oracle'))
print('roofline', d['roofline']); print('h2', d.get('h2')); print('cpu', d.get('cpu_baseline'), d.get('cpu_baseline_1core'))
print('clocks', d['clocks'], 'launches', d['gpu_launches'], d['details'].get('hierarchy'))
for s in d['sweeps']: print(s['level'], s['rows'], s['kernel'], s['sweep'][:8], round(s['ms']*1e3,1), 'us', round(s['gbs'],1))
"
tail -3 gpurun_out/r2z_b200_c3.err
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -4 | tee gpurun_out/r2z_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/r2z_smoke.log
