set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "modular or blocked or structures or vcycle or stream" 2>&1 | tail -4
python tools/sweep_tune.py c3 0 "lean_wpos=0" "lean_wpos=32" "lean_wpos=16" "lean_wpos=64;ring_bytes=24576" "lean_wpos=32;ring_bytes=24576" 2>&1 | grep level
python tools/sweep_tune.py c2 0 "lean_wpos=0" "lean_wpos=32" "lean_wpos=64;ring_bytes=24576" 2>&1 | grep level
python tools/sweep_tune.py c5 0 "lean_wpos=0" "lean_wpos=32" "lean_wpos=64;ring_bytes=24576" "lean_wpos=32;ring_bytes=24576" 2>&1 | grep level
