timeout 900 python -u -m pytest tests -x -q -m "gpu and not slow" -k "sparse or uniform or border or brick or approx or three_pass or golden or random_small or flag" --timeout 300 -p no:cacheprovider > gpurun_out/g16_tests.log 2>&1
tail -2 gpurun_out/g16_tests.log
python bench.py --runs c5_10 --no-e2e --no-cpu --no-small --no-work --detail --steps 5 > gpurun_out/g16_bench.json 2> gpurun_out/g16_bench.err
python tools/run_one.py c5_10 2 > gpurun_out/g16_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sp_border|sp_pairs" --csv --log-file /tmp/g16.csv python tools/run_one.py c5_10 1 > /dev/null 2>&1; cp /tmp/g16.csv gpurun_out/g16_k.csv
