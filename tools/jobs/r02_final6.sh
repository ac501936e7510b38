# round-2 evidence of HEAD: GPU suite, smoke, bench line (own + reference arm), launch list + full
# ncu capture of the squad kernel, per-config table, solve paths, C4 sweep, parity vs reference
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/r02_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/r02_smoke.log
timeout 600 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc $?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['closed_loop']['p50_tick_ms'], d['cpu_baseline']['value'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err; echo "ref rc $?"
bash tools/profile_round.sh r02n rti_squad_kernel 16384
timeout 900 python tools/configs.py > gpurun_out/r02_configs.json 2> gpurun_out/r02_configs.err; echo "configs rc $?"
timeout 900 python tools/paths.py > gpurun_out/r02_paths.jsonl 2> gpurun_out/r02_paths.err; echo "paths rc $?"
timeout 600 python tools/horizon_sweep.py 8192 > gpurun_out/r02_horizon_sweep.json 2> gpurun_out/r02_sweep.err; echo "sweep rc $?"
timeout 900 python tools/ref_parity.py gpurun_out/r02_ref_parity.json > gpurun_out/r02_ref_parity.log 2>&1; echo "ref_parity rc $?"
timeout 600 python tools/stress_determinism.py > gpurun_out/r02_stress_determinism.log 2>&1; echo "stress rc $?"
