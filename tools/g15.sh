timeout 600 python -u -m pytest tests -x -q -m gpu -k "brick or uniform_medium or sparse_and_csr" --timeout 300 -p no:cacheprovider > gpurun_out/g15_tests.log 2>&1
tail -2 gpurun_out/g15_tests.log
python bench.py --runs c5_10 --no-e2e --no-cpu --no-small --no-work --detail --steps 5 > gpurun_out/g15_bench.json 2> gpurun_out/g15_bench.err
