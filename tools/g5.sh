timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" > gpurun_out/g5_tests.log 2>&1
tail -3 gpurun_out/g5_tests.log
python bench.py --runs c5_10,c5_10k --no-e2e --no-cpu --detail --steps 5 > gpurun_out/g5_bench.json 2> gpurun_out/g5_bench.err
bash tools/prof.sh g5 c5_10 "sp_pairs|sp_border|lat_|sp_cells|label_roots|write_points" 14 0 "sp_pairs|sp_border_emit|lat_cells|lat_place|lat_count"
