# the per-agent kernel (warm start / sharing off / small batches) at C3 and its dense variant at N=5
python tools/ncu_driver.py 16384 10 2 0 > gpurun_out/r02j_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:rti_kernel -s 1 -c 1 -o gpurun_out/r02j_full python tools/ncu_driver.py 16384 10 2 0 > gpurun_out/r02j_ncu.log 2>&1; echo "j rc $?"
python tools/ncu_driver.py 8192 5 2 0 > gpurun_out/r02k_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:rti_kernel -s 1 -c 1 -o gpurun_out/r02k_full python tools/ncu_driver.py 8192 5 2 0 > gpurun_out/r02k_ncu.log 2>&1; echo "k rc $?"
