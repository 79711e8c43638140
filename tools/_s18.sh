set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "scan" > gpurun_out/s18_scan.log 2>&1; echo rc=$? >> gpurun_out/s18_scan.log
for sp in 0 16 64 256 100000000; do for sl in 0 32 100; do echo "spin=$sp sleep=$sl" >> gpurun_out/s18_probe.txt; MVAMG_SCAN_SPIN=$sp MVAMG_SCAN_SLEEP=$sl timeout 120 python tools/scan_probe.py c2 0 >> gpurun_out/s18_probe.txt 2>&1; done; done
