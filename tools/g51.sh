# c5 with the radix-sort grouping (F_RADIX_GROUP = 512): stage times and launch list
python tools/run_one.py c5_10 3 512 > gpurun_out/g51_plain.log 2>&1; tail -c 800 gpurun_out/g51_plain.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file /tmp/g51.csv python tools/run_one.py c5_10 1 512 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/g51.csv > gpurun_out/g51_launches.txt 2>&1; head -16 gpurun_out/g51_launches.txt
python tools/ncu_traffic.py /tmp/g51.csv 2>/dev/null | grep -i 'radix\|keys\|segment\|gather' | head
