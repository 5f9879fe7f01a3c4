# correctness of the new c5 kernels first, then timing
timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" > gpurun_out/g3_tests.log 2>&1
tail -5 gpurun_out/g3_tests.log
python bench.py --runs c5_10,c5_10k,c3 --no-e2e --no-cpu --detail --steps 5 > gpurun_out/g3_bench.json 2> gpurun_out/g3_bench.err
python tools/run_one.py c5_10 2 > gpurun_out/g3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/g3.csv python tools/run_one.py c5_10 1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/g3.csv > gpurun_out/g3_c5_launches.txt 2>&1
