set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_distributed.py -x -q -k "row or vcycle or pipelined or ipc or structures or fit_and_solve or stream or kcycle or composite" 2>&1 | tail -4
python tools/sweep_tune.py c3 1 "" 2>&1 | grep level
python tools/sweep_tune.py c3 3 "" 2>&1 | grep level
timeout 900 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-h2 > gpurun_out/r2g_b200_c3.json 2> gpurun_out/r2g_b200_c3.err
python -c "
import json; d=json.loads(open('gpurun_out/r2g_b200_c3.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'cycle', d['cycle']['ms'], 'nit', d['details']['nit'], d['roofline'])
for k in d['sweeps']: print(k['level'], k['kernel'], k['sweep'][:8], round(k['ms']*1e3,1), 'us')
"
python tools/sanitize_gs.py > gpurun_out/r2g_selfcheck.log 2>&1; tail -3 gpurun_out/r2g_selfcheck.log
