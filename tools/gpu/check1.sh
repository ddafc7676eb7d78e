# One-GPU regression check: GPU tests, smoke, GPT-2 and Llama-1B bench lines -> gpurun_out/c1/.
O=gpurun_out/c1; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 400 python bench.py > $O/bench_gpt2_n1.log 2>&1; echo "gpt2 n1 rc=$?"; tail -1 $O/bench_gpt2_n1.log
timeout 600 python bench.py --config llama-1b --batch 4 --seq 4096 --no-cpu-baseline > $O/bench_1b_n1.log 2>&1; echo "1b n1 rc=$?"; tail -1 $O/bench_1b_n1.log
