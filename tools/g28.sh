# list-based border: parity; ncu of the REC brick kernel
python -u -m pytest tests -x -q -m gpu -k "brick or border or c5_10 or sparse" --timeout 600 -p no:cacheprovider > gpurun_out/g28_tests.log 2>&1
tail -n 3 gpurun_out/g28_tests.log
bash tools/prof.sh g28 c5_10 "sp_core_brick|sp_border" 4 0 sp_core_brick; cat gpurun_out/g28_table.txt
