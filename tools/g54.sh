# lattice sort with compact 12-byte staging records: parity (lattice groupings, c5 full), c5 timing, launch list
python -u -m pytest tests -x -q -m gpu -k "lattice or brick or c5_10 or group or sparse or golden or random" --timeout 900 -p no:cacheprovider > gpurun_out/g54_tests.log 2>&1
tail -n 2 gpurun_out/g54_tests.log
python bench.py --runs c5_10,c5_10k --no-cpu --no-e2e --no-small --no-work --steps 10 > gpurun_out/g54_bench.json 2> gpurun_out/g54_bench.err
python -c "
import json;l=[x for x in open('gpurun_out/g54_bench.json') if x.startswith('{')][-1];d=json.loads(l)
for r in d.get('runs',[]): print(r['run'], r['ms_median'], r['stage_ms'])
"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lat_ --csv --log-file /tmp/g54.csv python tools/run_one.py c5_10 1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/g54.csv 2>&1 | head -10
