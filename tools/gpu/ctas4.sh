# GPT-2 W=4 step vs the NCCL CTA budget of the FSDP communicator.  bash tools/gpu/ctas4.sh
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29541"
for c in 0 2 4 8 16 0; do
  B2S_FSDP_MAX_CTAS=$c timeout 400 $TR --nproc-per-node 4 bench.py --gpus 4 --no-cpu-baseline --steps 20 > gpurun_out/c$c.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/c$c.log').read().strip().splitlines()[-1]); print('max_ctas=$c', d['ms_per_step'], d['e2e']['ms_per_step'], d['kernels']['gemm']['ms_per_step'], d['collectives']['reduce_scatter']['busbw_GBps'], d['clocks']['sm_mhz'])"
done
