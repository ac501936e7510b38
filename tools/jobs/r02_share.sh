timeout 600 python tools/share_check.py > gpurun_out/r02_share.log 2>&1; echo "share rc $?"
cat gpurun_out/r02_share.log
