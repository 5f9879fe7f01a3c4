#!/bin/bash
# Profile one BASELINE config on the GPU box and keep only TEXT summaries in
# gpurun_out/ (the .ncu-rep stays in /tmp: reports are too big to bring back).
# usage: tools/prof.sh NAME CONFIG KERNEL_REGEX COUNT [FLAGS]
set -u
name=$1; cfg=$2; rx=$3; cnt=$4; flags=${5:-0}
mkdir -p gpurun_out
python tools/run_one.py "$cfg" 1 "$flags" > "gpurun_out/${name}_plain.log" 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k "regex:$rx" -c "$cnt" -f -o "/tmp/$name" \
    python tools/run_one.py "$cfg" 1 "$flags" > "gpurun_out/${name}_ncu.log" 2>&1
python tools/ncu_table.py "/tmp/$name.ncu-rep" > "gpurun_out/${name}_table.txt" 2>&1
ncu -i "/tmp/$name.ncu-rep" --page raw --csv > "gpurun_out/${name}_raw.csv" 2>&1
ncu -i "/tmp/$name.ncu-rep" --page details > "gpurun_out/${name}_details.txt" 2>&1
# optional 6th argument: kernel-name regex whose per-source-line counters to export
if [ $# -ge 6 ]; then
  ncu -i "/tmp/$name.ncu-rep" --page source --csv --print-source sass --kernel-name "regex:$6" \
      > "gpurun_out/${name}_sass.csv" 2>&1
  ncu -i "/tmp/$name.ncu-rep" --page source --csv --print-source cuda --kernel-name "regex:$6" \
      > "gpurun_out/${name}_src.csv" 2>&1
  gzip -f "gpurun_out/${name}_sass.csv"
fi
