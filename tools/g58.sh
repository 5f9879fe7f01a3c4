# outputs allocated after the bounding-box launch: parity subset, small-call cost, bench
python -u -m pytest tests -x -q -m gpu -k "golden or random or abi or stream or host or c1 or c2" --timeout 900 -p no:cacheprovider > gpurun_out/g58_tests.log 2>&1
tail -n 2 gpurun_out/g58_tests.log
python tools/overhead.py > gpurun_out/g58_overhead.txt 2>&1; cat gpurun_out/g58_overhead.txt
python bench.py --no-cpu --no-e2e --no-work > gpurun_out/g58_bench.json 2> gpurun_out/g58_bench.err
python -c "
import json;l=[x for x in open('gpurun_out/g58_bench.json') if x.startswith('{')][-1];d=json.loads(l)
print(d['value'], d['ms_per_step'], [(r['run'], r['ms_median']) for r in d['runs']], d['small_config']['ms_median'])
"
