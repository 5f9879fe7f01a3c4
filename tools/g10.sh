python -u -m pytest tests -x -q -m "gpu and slow" --timeout 1500 -p no:cacheprovider > gpurun_out/g10_slow.log 2>&1
tail -3 gpurun_out/g10_slow.log
bash tools/prof.sh g10c5 c5_10 . 80
bash tools/prof.sh g10c3 c3 . 80
bash tools/prof.sh g10c47 c4_7d . 80
