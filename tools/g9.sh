python -u -m pytest tests -x -q -m "gpu and not slow" -k "brick or sparse or uniform or border or three_pass or golden or random_small or flag" --timeout 300 -p no:cacheprovider > gpurun_out/g9_tests.log 2>&1
tail -3 gpurun_out/g9_tests.log
python bench.py --runs c5_10,c3 --no-e2e --no-cpu --no-small --detail --steps 5 > gpurun_out/g9_bench.json 2> gpurun_out/g9_bench.err
bash tools/prof.sh g9 c5_10 "sp_core_brick" 1 0 "sp_core_brick"
