set -x
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" > gpurun_out/g1_lscpu.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
python tools/peak_dist.py > gpurun_out/g1_peak.jsonl 2> gpurun_out/g1_peak.err
timeout 1500 python -m pytest tests -x -q -m gpu -k "cell_tree_at_scale or three_pass or grouping_choice or overflow_falls or e2e_host_path_full" > gpurun_out/g1_tests.log 2>&1
python bench.py --no-cpu > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err
tail -3 gpurun_out/g1_tests.log
