# A/B of an env toggle on the GPT-2 step at W=1 and W=4 (same box). Usage: bash tools/gpu/ab4.sh VAR=VALUE
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29521"
for env in "X=0" "$1"; do
  env $env timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ab_1.log 2>&1
  env $env timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --no-cpu-baseline --steps 20 > gpurun_out/ab_4.log 2>&1
  for n in 1 4; do python -c "
import json
d=json.loads(open('gpurun_out/ab_$n.log').read().strip().splitlines()[-1])
print('$env', $n, d['ms_per_step'], d['tokens_per_sec_per_gpu'], {k: (v['ms_per_step'], v['tflops']) for k, v in d['kernels'].items()})"; done
done
