#!/bin/bash
# Launch list (every kernel with its device time) of one bench step, as text.
# usage: tools/launches.sh NAME [bench args...]
set -u
name=$1; shift
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-work "$@" > "gpurun_out/${name}_plain.log" 2>&1 || { echo "plain bench failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "/tmp/${name}.csv" \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-work "$@" > "gpurun_out/${name}_ncu.log" 2>&1
python tools/ncu_summary.py "/tmp/${name}.csv" > "gpurun_out/${name}_summary.txt" 2>&1
gzip -c "/tmp/${name}.csv" > "gpurun_out/${name}.csv.gz"
