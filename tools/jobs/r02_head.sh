# HEAD evidence: GPU suite, smoke, bench (own + reference arm), launch list, full ncu of the squad kernel
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/r02_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc $?"; cat gpurun_out/r02_smoke.log | tail -2
timeout 600 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc $?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'], d['roofline']['frac'], d.get('closed_loop',{}).get('p50_tick_ms'))"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err; echo "ref rc $?"
bash tools/profile_round.sh r02c rti_squad_kernel 16384
