O=gpurun_out/r2final4; mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest_all_4gpu.log 2>&1; echo pytest $?; tail -2 $O/pytest_all_4gpu.log
python bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_1b_n4.json 2> $O/bench_1b_n4.err; echo b1b4 $?
python bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_1b_n2.json 2> $O/bench_1b_n2.err; echo b1b2 $?
python bench.py --gpus 4 --config gpt2-124m --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_gpt2_n4.json 2> $O/bench_gpt2_n4.err; echo bg4 $?
python bench.py --gpus 4 --config llama-8b --steps 6 --warmup 3 --no-cpu-baseline > $O/bench_8b_n4.json 2> $O/bench_8b_n4.err; echo b8b $?
CUDA_VISIBLE_DEVICES=0 python bench.py --steps 20 --warmup 5 > $O/bench_1b_n1.json 2> $O/bench_1b_n1.err; echo b1b1 $?
