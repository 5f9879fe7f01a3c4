# c1 fixed cost: host timeline (DB_TRACE) and per-launch device times
DB_TRACE=1 python tools/run_one.py c1 3 > gpurun_out/g40_trace.log 2>&1
tail -n 60 gpurun_out/g40_trace.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/g40.csv python tools/run_one.py c1 1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/g40.csv > gpurun_out/g40_launches.txt 2>&1; cat gpurun_out/g40_launches.txt
python tools/overhead.py > gpurun_out/g40_overhead.txt 2>&1; cat gpurun_out/g40_overhead.txt
