# write_points: cells of > 32 core points by the whole warp; c1 fixed cost
python -u -m pytest tests -x -q -m gpu -k "golden or random or c1 or c5_10 or brick or sparse or label or determin" --timeout 900 -p no:cacheprovider > gpurun_out/g63_tests.log 2>&1
tail -n 2 gpurun_out/g63_tests.log
python tools/overhead.py 2>&1 | head -3
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:write_points --csv --log-file /tmp/g63.csv python tools/run_one.py c1 1 > /dev/null 2>&1; python tools/ncu_summary.py /tmp/g63.csv | head -3
