# checkpoint: all GPU tests, bench (coalesced scan stores, packed ClusterCore, lat_cells4)
python -u -m pytest tests -x -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/g44_tests.log 2>&1
tail -n 3 gpurun_out/g44_tests.log
python bench.py > gpurun_out/g44_bench.json 2> gpurun_out/g44_bench.err
python -c "
import json;l=[x for x in open('gpurun_out/g44_bench.json') if x.startswith('{')][-1];d=json.loads(l)
print(d['value'], d['ms_per_step'], json.dumps(d['roofline'])[:900])
for r in d.get('runs',[]): print(r['run'], r['ms_median'], r['stage_ms'])
"
