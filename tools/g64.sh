# row f2: query sub-cells one level finer (LQ = 9 / d): SS-simden 3D at large minPts
for mp in 3000 10000 30000; do python tools/run_pts.py ss 10000000 3 1000 $mp 2 2>&1 | tail -c 330; echo; done
python -u -m pytest tests -x -q -m gpu -k "subcell or qbound or flag" --timeout 900 -p no:cacheprovider > gpurun_out/g64_tests.log 2>&1
tail -n 2 gpurun_out/g64_tests.log
