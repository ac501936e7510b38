timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r02_pytest_gpu.log
timeout 300 python tools/squad_check.py --quick > gpurun_out/r02_q8_squad.log 2>&1; echo "squad_check rc $?"; grep "n=16384\|pair ==" gpurun_out/r02_q8_squad.log
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 60 --csv --log-file gpurun_out/r02_q8_launches_warm.csv python tools/ncu_driver.py 16384 10 3 > /dev/null 2>&1; echo "ncu rc $?"
