# Llama-8B (BASELINE configs[3]) FSDP steps on the GPUs of one box: W=4 with and
# without activation checkpointing, W=2 with it. Usage: bash tools/gpu/llama8b.sh
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29513"
nvidia-smi --query-gpu=name,memory.total --format=csv
for run in "4 --ac" "4" "2 --ac"; do
  set -- $run
  n=$1; shift
  tag="n${n}$(echo "$@" | tr -d ' -')"
  timeout 900 $TR --nproc-per-node $n bench.py --gpus $n --config llama-8b --batch 2 --seq 4096 --steps 5 \
      --warmup 3 --no-cpu-baseline "$@" > gpurun_out/bench_8b_$tag.log 2>&1
  echo "8b $tag rc=$?"; tail -c 700 gpurun_out/bench_8b_$tag.log; echo
done
