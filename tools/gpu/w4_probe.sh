# Where the W=4 GPT-2 step time goes: unit size and global-norm clipping variants (one 4-GPU box).
O=gpurun_out/w4p; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29541"
timeout 300 python bench.py --no-cpu-baseline > $O/n1.log 2>&1
for bpu in 1 2 4; do timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --no-cpu-baseline --blocks-per-unit $bpu > $O/n4_bpu$bpu.log 2>&1; done
B2S_GRAD_CLIP=0 timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --no-cpu-baseline > $O/n4_noclip.log 2>&1
timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --no-cpu-baseline > $O/n4_again.log 2>&1
for f in $O/*.log; do tail -1 $f | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$f'.split('/')[-1], d['ms_per_step'], d['value'])" 2>/dev/null || (echo "$f failed"; tail -3 $f); done
