# SS-varden 7D: ncu of the all-pairs neighbour search and its compaction
python tools/run_pts.py varden 10000000 7 2000 100 1 > gpurun_out/g72_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"nbr_brute|nbr_compact" -c 2 -f -o /tmp/g72 python tools/run_pts.py varden 10000000 7 2000 100 1 > gpurun_out/g72_ncu.log 2>&1
python tools/ncu_table.py /tmp/g72.ncu-rep > gpurun_out/g72_table.txt 2>&1; cat gpurun_out/g72_table.txt
ncu -i /tmp/g72.ncu-rep --page details > gpurun_out/g72_details.txt 2>&1
grep -E "Throughput|Eligible|Issued Warp|Occupancy|Registers|Executed Ipc|L2 Hit|L1/TEX Hit|Block Limit" gpurun_out/g72_details.txt | head -40
ncu -i /tmp/g72.ncu-rep --page source --csv --print-source sass --kernel-name regex:nbr_brute > gpurun_out/g72_sass.csv 2>&1; gzip -f gpurun_out/g72_sass.csv
python tools/sass_hot.py gpurun_out/g72_sass.csv.gz nbr_brute 16
