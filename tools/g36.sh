# ClusterCore on packed core points: parity, c5 timing, launch list
python -u -m pytest tests -x -q -m gpu -k "brick or border or c5_10 or sparse or packed or lattice or grouping or group" --timeout 600 -p no:cacheprovider > gpurun_out/g36_tests.log 2>&1
tail -n 5 gpurun_out/g36_tests.log
python bench.py --runs c5_10 --no-cpu --no-e2e --no-small --no-work > gpurun_out/g36_bench.json 2> gpurun_out/g36_bench.err
python -c "
import json;l=[x for x in open('gpurun_out/g36_bench.json') if x.startswith('{')][-1];d=json.loads(l)
print(d['ms_per_step'])
for r in d.get('runs',[]): print(r['run'], r['ms_median'], r['stage_ms'])
"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file /tmp/g36.csv python tools/run_one.py c5_10 1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/g36.csv > gpurun_out/g36_launches.txt 2>&1; head -40 gpurun_out/g36_launches.txt
