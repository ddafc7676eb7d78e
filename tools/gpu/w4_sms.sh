# W=4 GPT-2: persistent-GEMM SM budget vs NCCL CTA budget (one 4-GPU box).
O=gpurun_out/w4s; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29551"
run() { timeout 300 env "$@" $TR --nproc-per-node 4 bench.py --gpus 4 --no-cpu-baseline --blocks-per-unit 2 > $O/$(echo "$@" | tr ' =' '__').log 2>&1; }
run B2S_X=0
run B2S_GEMM_SMS=136
run B2S_GEMM_SMS=128
run B2S_GEMM_SMS=136 B2S_FSDP_MAX_CTAS=8
run B2S_GEMM_SMS=128 B2S_FSDP_MAX_CTAS=16
run B2S_X=1
for f in $O/*.log; do tail -1 $f | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$f'.split('/')[-1], d['ms_per_step'], d['value'])" 2>/dev/null || (echo "$f failed"; tail -3 $f); done
