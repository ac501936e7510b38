# z* contiguous-run output: full GPU suite + bench
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r02_zrun_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/r02_zrun_tests.log
timeout 600 python bench.py > gpurun_out/r02_zrun_bench.json 2> gpurun_out/r02_zrun_bench.err; echo "bench rc $?"
python -c "
import json;d=json.load(open('gpurun_out/r02_zrun_bench.json'));e=d['e2e']
print('device', d['ms_per_step'], 'e2e', e['ms_per_step'], 'noz', e['without_z_star']['ms_per_step'], 'soa', e['soa']['ms_per_step'], 'clocks', d.get('clocks'))"
