timeout 600 python tools/sq4_check.py > gpurun_out/r02_sq4.log 2>&1; echo "sq4 rc $?"; cat gpurun_out/r02_sq4.log | tail -30
