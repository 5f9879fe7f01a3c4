timeout 900 python -u -m pytest tests -x -q -m "gpu and not slow" --timeout 300 -p no:cacheprovider > gpurun_out/g12_tests.log 2>&1
tail -2 gpurun_out/g12_tests.log
python bench.py --no-cpu --no-e2e --detail > gpurun_out/g12_bench.json 2> gpurun_out/g12_bench.err
python tools/run_one.py c3 2 > gpurun_out/g12_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:group_ --csv --log-file /tmp/g12.csv python tools/run_one.py c4_7d 1 > /dev/null 2>&1; cp /tmp/g12.csv gpurun_out/g12_group.csv
