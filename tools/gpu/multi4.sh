set -x
nvidia-smi -L
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29511"
timeout 300 python -m pytest tests/test_fsdp_multigpu.py -m gpu -x -q > gpurun_out/w4_pytest_multi.log 2>&1; echo pytest=$?
for n in 2 4; do timeout 400 $TR --nproc-per-node $n bench.py --gpus $n --no-cpu-baseline > gpurun_out/w4_bench_gpt2_n$n.log 2>&1; echo bench$n=$?; done
timeout 600 python bench.py --config llama-1b --batch 4 --seq 4096 --no-cpu-baseline > gpurun_out/w4_bench_1b_n1.log 2>&1; echo b1=$?
timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --config llama-1b --batch 4 --seq 4096 --no-cpu-baseline > gpurun_out/w4_bench_1b_n4.log 2>&1; echo b14=$?
timeout 600 $TR --nproc-per-node 4 tools/collective_sweep.py gpurun_out/collective_sweep_w4.jsonl > gpurun_out/w4_sweep.log 2>&1; echo sweep=$?
for f in gpurun_out/w4_*.log; do echo == $f; tail -c 1500 $f; done
