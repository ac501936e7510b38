# quick kernel A/B: squad parity tests + C3 device time + stage split
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -x -k "parity_with_oracle or schedule_sharing or repeated or active_set" > gpurun_out/r02_quick_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/r02_quick_tests.log
timeout 300 python tools/squad_check.py --quick > gpurun_out/r02_quick_squad.log 2>&1; echo "squad_check rc $?"; tail -12 gpurun_out/r02_quick_squad.log
