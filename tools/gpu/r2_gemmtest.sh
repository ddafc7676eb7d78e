python -m pytest tests/test_gemm.py tests/test_guards.py tests/test_headline_parity.py -m gpu -q -x -k "gemm or swiglu or rope or two_layer or guard or bounds" 2>&1 | tail -3
python tools/bench_kernels.py 2>/dev/null | grep -i "llama\|swiglu"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_gemm.json 2>/dev/null; echo bench $?
