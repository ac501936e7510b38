timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_parity.py -q -rf -x > gpurun_out/r02_q9_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/r02_q9_tests.log
timeout 300 python tools/squad_check.py --quick > gpurun_out/r02_q9_squad.log 2>&1; echo "squad_check rc $?"; grep "n=16384\|squad vs oracle" gpurun_out/r02_q9_squad.log
