timeout 600 python -u -m pytest tests -x -q -m gpu -k "approx" --timeout 300 -p no:cacheprovider > gpurun_out/g11_tests.log 2>&1
tail -2 gpurun_out/g11_tests.log
python tools/sweep.py --only approx --reps 2 > gpurun_out/g11_approx.jsonl 2> gpurun_out/g11_approx.err
python bench.py --no-cpu > gpurun_out/g11_bench.json 2> gpurun_out/g11_bench.err
