# final round-2 evidence: the driver's order (reference arm first, then the B200 arm), GPU suite, smoke
set -x
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -6 | tee gpurun_out/r2z_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/r2z_smoke.log
timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2z_ref_c3.json 2> gpurun_out/r2z_ref_c3.err
tail -c 1500 gpurun_out/r2z_ref_c3.json
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r2z_b200_c3.json 2> gpurun_out/r2z_b200_c3.err
python -c "
import json; d=json.loads(open('gpurun_out/r2z_b200_c3.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'cycle', d['cycle']['ms'], 'nit', d['details']['nit'])
print('roofline', d['roofline']); print('h2', d.get('h2')); print('cpu', d.get('cpu_baseline'), d.get('cpu_baseline_1core'))
print('clocks', d['clocks'], 'launches', d['gpu_launches'])
"
tail -3 gpurun_out/r2z_b200_c3.err
