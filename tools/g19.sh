python tools/run_pts.py varden 10000000 7 2000 100 2 > gpurun_out/g19_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed_per_inst_executed.ratio --clock-control none --csv --log-file /tmp/g19.csv python tools/run_pts.py varden 10000000 7 2000 100 1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/g19.csv > gpurun_out/g19_launches.txt 2>&1; cp /tmp/g19.csv gpurun_out/g19.csv
