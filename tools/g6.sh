timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" > gpurun_out/g6_tests.log 2>&1
tail -3 gpurun_out/g6_tests.log
python bench.py --no-cpu --detail > gpurun_out/g6_bench.json 2> gpurun_out/g6_bench.err
DB_TRACE=1 python tools/run_one.py c3 3 > gpurun_out/g6_trace_c3.txt 2>&1
DB_TRACE=1 python tools/run_one.py c5_10 3 > gpurun_out/g6_trace_c5.txt 2>&1
python tools/run_one.py c5_10 2 > gpurun_out/g6_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/g6.csv python tools/run_one.py c5_10 1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/g6.csv > gpurun_out/g6_c5_launches.txt 2>&1
