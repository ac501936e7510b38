timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -q -rf -x > gpurun_out/r02_q2_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/r02_q2_tests.log
timeout 300 python tools/squad_check.py --quick > gpurun_out/r02_q2_squad.log 2>&1; echo "squad_check rc $?"; tail -2 gpurun_out/r02_q2_squad.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02_q2_launches.csv python tools/ncu_driver.py 16384 10 3 > /dev/null 2>&1; echo "ncu rc $?"
