# sub-cell stencil brick MarkCore: parity (brick tests + full c5) and c5 timing
python -u -m pytest tests -x -q -m gpu -k "brick or border_c5 or c5_10" --timeout 600 -p no:cacheprovider > gpurun_out/g21_tests.log 2>&1
tail -n 3 gpurun_out/g21_tests.log
python bench.py --runs c5_10 --no-cpu --no-e2e --no-small --detail > gpurun_out/g21_bench.json 2> gpurun_out/g21_bench.err
python -c "
import json;l=[x for x in open('gpurun_out/g21_bench.json') if x.startswith('{')][-1];d=json.loads(l)
print(d['ms_per_step'], json.dumps(d['roofline'])[:400])
for r in d.get('runs',[]): print(r['run'], r['ms_median'], r['stage_ms'])
"
tail -n 5 gpurun_out/g21_bench.err
