# brick MarkCore: sub-cell stencils (padded rows) + 16-bit halo-relative points
python -u -m pytest tests -x -q -m gpu -k "brick or border_c5 or c5_10 or sparse" --timeout 600 -p no:cacheprovider > gpurun_out/g24_tests.log 2>&1
tail -n 3 gpurun_out/g24_tests.log
python bench.py --runs c5_10 --no-cpu --no-e2e --no-small > gpurun_out/g24_bench.json 2> gpurun_out/g24_bench.err
python -c "
import json;l=[x for x in open('gpurun_out/g24_bench.json') if x.startswith('{')][-1];d=json.loads(l)
print(d['ms_per_step'], json.dumps(d['roofline'])[:300])
for r in d.get('runs',[]): print(r['run'], r['ms_median'], r['stage_ms'])
"
bash tools/prof.sh g24 c5_10 sp_core_brick 1 0 sp_core_brick; cat gpurun_out/g24_table.txt
