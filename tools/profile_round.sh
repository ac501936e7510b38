#!/bin/bash
# Run ON the GPU box (gpurun): the ncu evidence for profiles/.  Each ncu command runs only
# after the same command exited 0 without ncu.
#   1. launch list of the bench command (per-launch gpu__time_duration, serialised, cold cache)
#   2. one full-set capture of the solve kernel at the bench workload (DRAM traffic, stalls)
set -e
tag=${1:-r01}
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_plain_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${tag}_ncu_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${tag}_ncu_bench.log 2>&1
python tools/ncu_driver.py 4096 10 2
ncu --set full --import-source on --clock-control none -k regex:rti_kernel -c 1 \
    -o gpurun_out/${tag}_full python tools/ncu_driver.py 4096 10 2 > gpurun_out/${tag}_ncu_full.log 2>&1
echo done
