#!/bin/bash
# usage: prof_pts.sh NAME KREGEX COUNT args-for-run_pts...
name=$1; rx=$2; cnt=$3; shift 3
ncu --set full --clock-control none --import-source on -k "regex:$rx" -c "$cnt" -f -o "/tmp/$name" python tools/run_pts.py "$@" > "gpurun_out/${name}_ncu.log" 2>&1
python tools/ncu_table.py "/tmp/$name.ncu-rep" > "gpurun_out/${name}_table.txt" 2>&1
ncu -i "/tmp/$name.ncu-rep" --page details > "gpurun_out/${name}_details.txt" 2>&1
ncu -i "/tmp/$name.ncu-rep" --page source --csv --print-source sass > "gpurun_out/${name}_sass.csv" 2>&1
gzip -f "gpurun_out/${name}_sass.csv"
