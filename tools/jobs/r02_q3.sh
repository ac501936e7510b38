timeout 1200 python -m pytest tests/test_gpu_parity.py -q -rf -x -k "parity_with_oracle or schedule_sharing or repeated or active_set or auto" > gpurun_out/r02_q3_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/r02_q3_tests.log
timeout 300 python tools/squad_check.py --quick > gpurun_out/r02_q3_squad.log 2>&1; echo "squad_check rc $?"; cat gpurun_out/r02_q3_squad.log | grep -v "^  pair"
