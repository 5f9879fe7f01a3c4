timeout 900 python -u -m pytest tests -x -q -m gpu -k "three_axis or clustered_medium or varden or cell_tree" --timeout 600 -p no:cacheprovider > gpurun_out/g14_tests.log 2>&1
tail -2 gpurun_out/g14_tests.log
python tools/sweep.py --only varden --reps 2 > gpurun_out/g14_varden.jsonl 2> gpurun_out/g14_varden.err
python tools/sweep.py --only eps --reps 2 > gpurun_out/g14_eps.jsonl 2> gpurun_out/g14_eps.err
python tools/sweep.py --only minpts --reps 2 > gpurun_out/g14_minpts.jsonl 2> gpurun_out/g14_minpts.err
