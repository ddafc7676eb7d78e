O=gpurun_out/r2multi; mkdir -p $O
nvidia-smi -L > $O/gpus.txt
python -m pytest tests/test_fsdp_multigpu.py -m gpu -v -x > $O/pytest_multigpu_w4.log 2>&1; echo multi $?
python bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_1b_n4.json 2> $O/bench_1b_n4.err; echo bench4 $?
python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_1b_n2.json 2> $O/bench_1b_n2.err; echo bench2 $?
