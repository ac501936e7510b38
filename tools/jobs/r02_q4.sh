timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r02_pytest_gpu.log
timeout 300 python tools/squad_check.py --quick > gpurun_out/r02_q4_squad.log 2>&1; echo "squad_check rc $?"; grep "n=16384" gpurun_out/r02_q4_squad.log
bash tools/profile_round.sh r02d rti_squad_kernel 16384
