# final-state check (3): all GPU tests, smoke, default bench
python -u -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/g79_tests.log 2>&1
tail -n 3 gpurun_out/g79_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g79_smoke.log 2>&1; tail -n 1 gpurun_out/g79_smoke.log
python bench.py > gpurun_out/g79_bench.json 2> gpurun_out/g79_bench.err
python -c "
import json;l=[x for x in open('gpurun_out/g79_bench.json') if x.startswith('{')][-1];d=json.loads(l)
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('executed_frac'), d['e2e']['value'], d['clocks'])
"
