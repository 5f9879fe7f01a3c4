# hash grouping: a warp's chunk loaded before its steps (8 or 4 x 32 points in flight)
python -u -m pytest tests -x -q -m gpu -k "group or c1 or c2 or varden or golden or random or full_config" --timeout 900 -p no:cacheprovider > gpurun_out/g42_tests.log 2>&1
tail -n 2 gpurun_out/g42_tests.log
python bench.py --runs c2,c3,c4_5d,c4_7d --no-cpu --no-e2e --no-small --no-work --steps 10 > gpurun_out/g42_bench.json 2> gpurun_out/g42_bench.err
python -c "
import json;l=[x for x in open('gpurun_out/g42_bench.json') if x.startswith('{')][-1];d=json.loads(l)
for r in d.get('runs',[]): print(r['run'], r['ms_median'], r['stage_ms'])
"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:group_ --csv --log-file /tmp/g42.csv python tools/run_one.py c3 1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/g42.csv | head -8
