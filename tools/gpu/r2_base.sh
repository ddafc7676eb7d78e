set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/r2b_pytest.log 2>&1; echo pytest rc $?
python bench.py --config llama-1b --batch 4 --seq 4096 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench_1b.json 2> gpurun_out/r2b_bench_1b.err; echo rc $?
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench_gpt2.json 2> gpurun_out/r2b_bench_gpt2.err; echo rc $?
