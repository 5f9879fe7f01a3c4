# all-pairs neighbour search: own entries forward without atomics, mirror entries backward
python -u -m pytest tests -x -q -m gpu -k "varden or tree or nbr or two_pass or dim or random or c4 or approx or flag" --timeout 900 -p no:cacheprovider > gpurun_out/g75_tests.log 2>&1
tail -n 2 gpurun_out/g75_tests.log
python tools/run_pts.py varden 10000000 7 2000 100 2 2>&1 | tail -c 250
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"nbr_" --csv --log-file /tmp/g75.csv python tools/run_pts.py varden 10000000 7 2000 100 1 > /dev/null 2>&1; python tools/ncu_summary.py /tmp/g75.csv | head -5
