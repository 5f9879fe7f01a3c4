# host timelines (DB_TRACE) of c3 and c5_10: where the GPU waits for the host
DB_TRACE=1 python tools/run_one.py c3 2 > gpurun_out/g52_c3.log 2>&1
DB_TRACE=1 python tools/run_one.py c5_10 2 > gpurun_out/g52_c5.log 2>&1
DB_TRACE=1 python tools/run_one.py c2 2 > gpurun_out/g52_c2.log 2>&1
