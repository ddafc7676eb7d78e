# GPT-2 W=4 step under NCCL channel / NVLS settings (how much do the collectives slow the compute?).
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29517"
for env in "X=1" "NCCL_MAX_NCHANNELS=2" "NCCL_MAX_NCHANNELS=8" "NCCL_NVLS_ENABLE=0" "NCCL_NVLS_ENABLE=1 NCCL_MAX_NCHANNELS=2"; do
  env $env timeout 400 $TR --nproc-per-node 4 bench.py --gpus 4 --no-cpu-baseline --steps 20 > gpurun_out/nccl_$$.log 2>&1
  python -c "
import json,sys
d=json.loads(open('gpurun_out/nccl_$$.log').read().strip().splitlines()[-1])
print('$env', d['ms_per_step'], d['tokens_per_sec_per_gpu'], d['kernels']['gemm']['ms_per_step'], d['e2e']['ms_per_step'])"
done
NCCL_DEBUG=INFO timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --no-cpu-baseline --steps 3 2>&1 | grep -iE "nvls|channel|algo|proto" | head -20
