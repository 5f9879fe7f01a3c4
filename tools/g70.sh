# grouping: 32-bit multiply-high cell division; parity and bench
python -u -m pytest tests -x -q -m gpu -k "golden or random or group or lattice or flag or c1 or c2 or full_config or extreme or edge or dim" --timeout 900 -p no:cacheprovider > gpurun_out/g70_tests.log 2>&1
tail -n 2 gpurun_out/g70_tests.log
python bench.py --no-cpu --no-e2e --no-work > gpurun_out/g70_bench.json 2> gpurun_out/g70_bench.err
python -c "
import json;l=[x for x in open('gpurun_out/g70_bench.json') if x.startswith('{')][-1];d=json.loads(l)
print(d['value'], d['ms_per_step'], [(r['run'], r['ms_median'], r['stage_ms'].get('keys+sort')) for r in d['runs']])
"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"group_|lat_" --csv --log-file /tmp/g70.csv python tools/run_one.py c3 1 > /dev/null 2>&1; python tools/ncu_summary.py /tmp/g70.csv | head -6
