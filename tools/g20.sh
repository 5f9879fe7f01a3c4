# Round-2 re-entry check: all GPU tests (incl. full-size slow parity), smoke, bench.
python -u -m pytest tests -x -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/g20_tests.log 2>&1
tail -n 5 gpurun_out/g20_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g20_smoke.log 2>&1; tail -n 2 gpurun_out/g20_smoke.log
python bench.py > gpurun_out/g20_bench.json 2> gpurun_out/g20_bench.err; tail -c 3000 gpurun_out/g20_bench.json
