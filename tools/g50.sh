# brick MarkCore, 3 CTAs per SM: 384 threads, thread copies instead of TMA, 16-bit window lists
python -u -m pytest tests -x -q -m gpu -k "brick or c5_10" --timeout 600 -p no:cacheprovider > gpurun_out/g50_tests.log 2>&1
tail -n 2 gpurun_out/g50_tests.log
python bench.py --runs c5_10 --no-cpu --no-e2e --no-small --no-work --steps 10 > gpurun_out/g50_bench.json 2> gpurun_out/g50_bench.err
python -c "
import json;l=[x for x in open('gpurun_out/g50_bench.json') if x.startswith('{')][-1];d=json.loads(l)
for r in d.get('runs',[]): print(r['run'], r['ms_median'], r['stage_ms'])
"
