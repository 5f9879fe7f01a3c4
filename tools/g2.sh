python bench.py --no-cpu --detail > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err
timeout 2400 python tools/cpu_baselines.py > gpurun_out/g2_cpu.jsonl 2> gpurun_out/g2_cpu.err
