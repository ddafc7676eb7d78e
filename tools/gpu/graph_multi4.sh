# W>1 CUDA graph (default on): 2-GPU parity tests, W=2 / W=4 bench with the graph on and off.
O=gpurun_out/gm4; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29591"
timeout 400 python -m pytest tests/test_fsdp_multigpu.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for n in 2 4; do for r in 1 2; do
  B2S_GRAPH_MULTI=1 timeout 300 $TR --nproc-per-node $n bench.py --gpus $n --no-cpu-baseline > $O/on_n${n}_$r.log 2>&1; echo "on n$n rc=$?"
  B2S_GRAPH_MULTI=0 timeout 300 $TR --nproc-per-node $n bench.py --gpus $n --no-cpu-baseline > $O/off_n${n}_$r.log 2>&1
done; done
timeout 300 python bench.py --no-cpu-baseline > $O/n1.log 2>&1
for f in $O/*.log; do tail -1 $f | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$f'.split('/')[-1], d['ms_per_step'], d['value'], d['e2e']['value'])" 2>/dev/null; done
