# SS-varden 7D: stage times and launch list on the current build
python tools/run_pts.py varden 10000000 7 2000 100 3 > gpurun_out/g43_plain.log 2>&1; tail -c 1500 gpurun_out/g43_plain.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file /tmp/g43.csv python tools/run_pts.py varden 10000000 7 2000 100 1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/g43.csv > gpurun_out/g43_launches.txt 2>&1; head -30 gpurun_out/g43_launches.txt
