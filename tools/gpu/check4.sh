# Kernel tests + multi-GPU equivalence + GPT-2 bench at W=1,2,4 (one 4-GPU box).
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29519"
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/c4_n1.log 2>&1
for n in 2 4; do timeout 300 $TR --nproc-per-node $n bench.py --gpus $n --no-cpu-baseline --steps 20 > gpurun_out/c4_n$n.log 2>&1; done
for n in 1 2 4; do python -c "
import json
d=json.loads(open('gpurun_out/c4_n$n.log').read().strip().splitlines()[-1])
print($n, d['ms_per_step'], d['tokens_per_sec_per_gpu'], d['mfu'], {k: (v['ms_per_step'], v['tflops']) for k, v in d['kernels'].items()}, d['e2e']['ms_per_step'])"; done
