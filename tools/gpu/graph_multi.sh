# W>1 CUDA-graph path: parity (2-GPU tests with the graph on) and timing, same box.
O=gpurun_out/gm; mkdir -p $O
N=${1:-2}
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29561"
B2S_GRAPH_MULTI=1 timeout 400 python -m pytest tests/test_fsdp_multigpu.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
for r in 1 2; do
  B2S_GRAPH_MULTI=0 timeout 300 $TR --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline > $O/off_$r.log 2>&1
  B2S_GRAPH_MULTI=1 timeout 300 $TR --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline > $O/on_$r.log 2>&1
done
for f in $O/*_?.log; do tail -1 $f | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$f'.split('/')[-1], d['ms_per_step'], d['value'], d['e2e']['value'])" 2>/dev/null || (echo "$f failed"; tail -5 $f); done
