# warp-cooperative core counts of large non-dense cells: parity subset, minPts 3e4 instance
python -u -m pytest tests -x -q -m gpu -k "subcell or qbound or golden or random or flag or c3 or varden" --timeout 900 -p no:cacheprovider > gpurun_out/g61_tests.log 2>&1
tail -n 2 gpurun_out/g61_tests.log
python tools/run_pts.py ss 10000000 3 1000 30000 2 2>&1 | tail -c 300
