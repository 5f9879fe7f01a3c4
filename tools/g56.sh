# compute-sanitizer on small instances (c1 and a c5-like sparse lattice)
timeout 300 compute-sanitizer --tool memcheck --print-limit 20 python tools/run_one.py c1 1 > gpurun_out/g56_memcheck_c1.txt 2>&1; echo "memcheck c1 rc=$?"
tail -n 5 gpurun_out/g56_memcheck_c1.txt
timeout 300 compute-sanitizer --tool memcheck --print-limit 20 python tools/run_pts.py uniform 200000 3 2500 10 1 > gpurun_out/g56_memcheck_sparse.txt 2>&1; echo "memcheck sparse rc=$?"
tail -n 5 gpurun_out/g56_memcheck_sparse.txt
