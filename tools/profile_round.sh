#!/bin/bash
# Run ON the GPU box (gpurun): the ncu evidence for profiles/.  Each ncu command runs only
# after the same command exited 0 without ncu.
#   1. launch list of the bench command (per-launch gpu__time_duration, serialised, cold cache)
#   2. one full-set capture of the solve kernel at the bench workload (C3: 16 384 agents, N=10)
tag=${1:-r02}
kern=${2:-rti_shared_kernel}
n=${3:-16384}
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ppo --cl-agents 0 > gpurun_out/${tag}_plain_bench.json 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/${tag}_ncu_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ppo --cl-agents 0 \
    > gpurun_out/${tag}_ncu_bench.log 2>&1
echo "launch list rc $?"
python tools/ncu_driver.py $n 10 2 > gpurun_out/${tag}_driver_plain.log 2>&1 &&
ncu --set full --import-source on --clock-control none -k regex:$kern -s 1 -c 1 \
    -o gpurun_out/${tag}_full python tools/ncu_driver.py $n 10 2 > gpurun_out/${tag}_ncu_full.log 2>&1
echo "full rc $?"
