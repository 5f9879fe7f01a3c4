# brick MarkCore with 18^3 bricks (halo replication 1.83 instead of 1.95)
python -u -m pytest tests -x -q -m gpu -k "brick or c5_10 or sparse or packed or border" --timeout 600 -p no:cacheprovider > gpurun_out/g83_tests.log 2>&1
tail -n 2 gpurun_out/g83_tests.log
python bench.py --runs c5_10 --no-cpu --no-e2e --no-small --no-work --steps 10 > gpurun_out/g83_bench.json 2> gpurun_out/g83_bench.err
python -c "
import json;l=[x for x in open('gpurun_out/g83_bench.json') if x.startswith('{')][-1];d=json.loads(l)
for r in d.get('runs',[]): print(r['run'], r['ms_median'], r['stage_ms'])
"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sp_core_brick|sp_cells" --csv --log-file /tmp/g83.csv python tools/run_one.py c5_10 1 > /dev/null 2>&1; python tools/ncu_summary.py /tmp/g83.csv | head -4
