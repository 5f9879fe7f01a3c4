# SS-varden 7D: ClusterCore kernels (waves, large BCPs)
ncu --metrics gpu__time_duration.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum --clock-control none -k regex:"wave_csr|bcp_large|uf_|mark_core" --csv --log-file /tmp/g76.csv python tools/run_pts.py varden 10000000 7 2000 100 1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/g76.csv | head -20
python tools/ncu_traffic.py /tmp/g76.csv 2>/dev/null | head -20
