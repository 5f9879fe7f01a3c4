python -u -m pytest tests -x -q -m "gpu and not slow" --timeout 300 -p no:cacheprovider > gpurun_out/g8_tests.log 2>&1
tail -3 gpurun_out/g8_tests.log
python bench.py --no-cpu --detail > gpurun_out/g8_bench.json 2> gpurun_out/g8_bench.err
DB_TRACE=1 python tools/run_one.py c3 3 > gpurun_out/g8_trace_c3.txt 2>&1
python tools/overhead.py > gpurun_out/g8_overhead.txt 2>&1
