timeout 900 python -u -m pytest tests -x -q -m "gpu and not slow" --timeout 300 -p no:cacheprovider > gpurun_out/g17_tests.log 2>&1
tail -2 gpurun_out/g17_tests.log
python bench.py --no-cpu --no-e2e --detail > gpurun_out/g17_bench.json 2> gpurun_out/g17_bench.err
python tools/overhead.py > gpurun_out/g17_overhead.txt 2>&1
