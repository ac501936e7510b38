ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 60 --csv --log-file gpurun_out/r02_q7_launches_warm.csv python tools/ncu_driver.py 16384 10 3 > /dev/null 2>&1; echo "ncu rc $?"
python tools/latency_split.py 10 2>&1 | tail -3
