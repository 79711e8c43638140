set -x
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1c_c2_launches.csv python tools/profile_solve.py c2 solve > gpurun_out/r1c_ncu_launch.log 2>&1
