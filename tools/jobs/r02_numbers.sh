timeout 600 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc $?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['closed_loop']['p50_tick_ms'], d['cpu_baseline']['value'])"
timeout 600 python tools/horizon_sweep.py 8192 > gpurun_out/r02_horizon_sweep.json 2> gpurun_out/r02_sweep.err; echo "sweep rc $?"
python -c "import json; d=json.load(open('gpurun_out/r02_horizon_sweep.json')); [print(r['horizon'], r['ms_per_tick_p50'], r['roofline_frac']) for r in d['rows']]"
timeout 900 python tools/paths.py > gpurun_out/r02_paths.jsonl 2> gpurun_out/r02_paths.err; echo "paths rc $?"; cat gpurun_out/r02_paths.jsonl
