O=gpurun_out/r2multi4b; mkdir -p $O
python bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_1b_n4.json 2> $O/bench_1b_n4.err; echo b1b $?
python bench.py --gpus 4 --config gpt2-124m --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_gpt2_n4.json 2> $O/bench_gpt2_n4.err; echo bgpt2 $?
python bench.py --gpus 4 --config llama-8b --steps 6 --warmup 3 --no-cpu-baseline > $O/bench_8b_n4.json 2> $O/bench_8b_n4.err; echo b8b $?
python bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_1b_n2.json 2> $O/bench_1b_n2.err; echo b1b2 $?
