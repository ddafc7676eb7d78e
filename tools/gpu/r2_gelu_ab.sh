for i in 1 2; do
python bench.py --config gpt2-124m --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('base', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['kernels']['gemm'])"
B2S_LIB=paper_2602_08387_b200/csrc/build/var_gelu8/libb2s.so python bench.py --config gpt2-124m --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gelu8', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['kernels']['gemm'])"
done
