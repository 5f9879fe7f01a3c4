python -u -m pytest tests -x -v -m "gpu and not slow" --timeout 300 -p no:cacheprovider > gpurun_out/g7_tests.log 2>&1
tail -5 gpurun_out/g7_tests.log
python tools/sweep.py --only qt --reps 2 > gpurun_out/g7_qt.jsonl 2> gpurun_out/g7_qt.err
