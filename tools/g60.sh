# warp-cooperative stable partition of large mixed cells: parity, minPts sweep (compact stage), bench
python -u -m pytest tests -x -q -m gpu -k "subcell or qbound or golden or random or flag or c5_10 or brick or sparse or full_config" --timeout 900 -p no:cacheprovider > gpurun_out/g60_tests.log 2>&1
tail -n 2 gpurun_out/g60_tests.log
python tools/sweep.py --reps 2 --only minpts > gpurun_out/g60_minpts.jsonl 2>/dev/null
python -c "
import json
for l in open('gpurun_out/g60_minpts.jsonl'):
    d=json.loads(l); print(d['data'], d['min_pts'], d['ms'], {k:d['stage_ms'][k] for k in ('markcore','compact','border') if k in d['stage_ms']})
"
python bench.py --no-cpu --no-e2e --no-work > gpurun_out/g60_bench.json 2> gpurun_out/g60_bench.err
python -c "
import json;l=[x for x in open('gpurun_out/g60_bench.json') if x.startswith('{')][-1];d=json.loads(l)
print(d['value'], d['ms_per_step'], [(r['run'], r['ms_median'], r['stage_ms'].get('compact')) for r in d['runs']])
"
