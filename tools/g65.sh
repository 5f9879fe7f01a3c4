# U1 variant 3 (the brick predicate): peaks, and the bench line with it as the MarkCore denominator
python -c "
import paper_1912_06255_b200 as pkg
for v in (0, 3):
    for qt in (1, 2, 4):
        r = pkg.peak_dist(3, v, qt, reps=60); print(v, qt, round(r['tests_per_s']/1e12, 3))
"
python bench.py --no-e2e --no-cpu --runs c5_10 > gpurun_out/g65_bench.json 2> gpurun_out/g65_bench.err
python -c "
import json;l=[x for x in open('gpurun_out/g65_bench.json') if x.startswith('{')][-1];d=json.loads(l)
print(json.dumps(d['roofline'])[:700]); print(d.get('peaks_u1'))
"
