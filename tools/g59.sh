# rows f1, f2, f4 sweeps on the final round-2 build
python tools/sweep.py --reps 3 > gpurun_out/r2b_sweeps.jsonl 2> gpurun_out/r2b_sweeps.err
wc -l gpurun_out/r2b_sweeps.jsonl; tail -n 3 gpurun_out/r2b_sweeps.err
