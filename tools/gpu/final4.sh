# Full measurement set on one 4-GPU box: tests, GPT-2 at W=1/2/4, Llama-1B at W=1/4, Llama-8B (AC) at W=4,
# the W=4 collective sweep. Outputs in gpurun_out/final/.   bash tools/gpu/final4.sh
O=gpurun_out/final; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29531"
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 400 python bench.py > $O/bench_gpt2_n1.log 2>&1; echo "gpt2 n1 rc=$?"
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.log 2>&1; echo "ref rc=$?"
for n in 2 4; do timeout 400 $TR --nproc-per-node $n bench.py --gpus $n > $O/bench_gpt2_n$n.log 2>&1; echo "gpt2 n$n rc=$?"; done
timeout 600 python bench.py --config llama-1b --batch 4 --seq 4096 --no-cpu-baseline > $O/bench_1b_n1.log 2>&1; echo "1b n1 rc=$?"
timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --config llama-1b --batch 4 --seq 4096 > $O/bench_1b_n4.log 2>&1; echo "1b n4 rc=$?"
timeout 900 $TR --nproc-per-node 4 bench.py --gpus 4 --config llama-8b --batch 2 --seq 4096 --ac --steps 5 > $O/bench_8b_n4ac.log 2>&1; echo "8b n4 rc=$?"
for f in $O/bench_*.log; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f.split("/")[-1], d.get("n_gpus"), d.get("ms_per_step"), d.get("tokens_per_sec_per_gpu"), d.get("mfu"),
          (d.get("e2e") or {}).get("value"), (d.get("roofline") or {}).get("frac"), d.get("clocks"))
except Exception as e:
    print(f, "unparsed", e)
PY
done
