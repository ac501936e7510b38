# the store build (rti_kernel mode 1, one CTA per schedule) at C3: full-set capture for stall attribution
python tools/ncu_driver.py 16384 10 3 > gpurun_out/r02g_plain.log 2>&1; echo "plain rc $?"
ncu --set full --import-source on --clock-control none -k regex:rti_kernel -s 2 -c 1 -o gpurun_out/r02g_store python tools/ncu_driver.py 16384 10 3 > gpurun_out/r02g_ncu.log 2>&1; echo "ncu rc $?"
