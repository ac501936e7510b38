timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r02_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 300 python tools/squad_check.py --quick > gpurun_out/r02_q6_squad.log 2>&1; echo "squad_check rc $?"; grep "n=16384" gpurun_out/r02_q6_squad.log
timeout 600 python bench.py --no-ppo --no-cpu-baseline > gpurun_out/r02_q6_bench.json 2>gpurun_out/r02_q6_bench.err; echo "bench rc $?"
python -c "import json; d=json.load(open('gpurun_out/r02_q6_bench.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'], d['gpu_launches'], d['closed_loop'])"
timeout 300 torchrun --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 5 --warmup 3 --no-ppo --no-cpu-baseline --cl-agents 0 > gpurun_out/r02_q6_torchrun.json 2> gpurun_out/r02_q6_torchrun.err; echo "torchrun rc $?"; tail -c 300 gpurun_out/r02_q6_torchrun.json
