# brick MarkCore with a preferred shared-memory carveout of 86% (196 KB: two CTAs, the rest L1)
python bench.py --runs c5_10 --no-cpu --no-e2e --no-small --no-work --steps 10 > gpurun_out/g84_bench.json 2> gpurun_out/g84_bench.err
python -c "
import json;l=[x for x in open('gpurun_out/g84_bench.json') if x.startswith('{')][-1];d=json.loads(l)
for r in d.get('runs',[]): print(r['run'], r['ms_median'], r['stage_ms'])
"
ncu --metrics gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:sp_core_brick --csv --log-file /tmp/g84.csv python tools/run_one.py c5_10 1 > /dev/null 2>&1; grep -v '^==' /tmp/g84.csv | tail -3
ncu --set full --clock-control none -k regex:sp_core_brick -c 1 python tools/run_one.py c5_10 1 2>/dev/null | grep -E 'Shared Memory Configuration Size|L1/TEX Hit Rate|Duration' | head -5
