# per-kernel device times (ncu, cold) of c2 and c1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/g53a.csv python tools/run_one.py c2 1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/g53a.csv > gpurun_out/g53_c2.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/g53b.csv python tools/run_one.py c1 1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/g53b.csv > gpurun_out/g53_c1.txt 2>&1
cat gpurun_out/g53_c2.txt
