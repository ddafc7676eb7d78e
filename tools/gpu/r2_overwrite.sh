O=gpurun_out/r2ow; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo pytest $?; tail -2 $O/pytest.log
for i in 1 2; do
python bench.py --steps 20 --warmup 4 --no-cpu-baseline > $O/b_$i.json 2>/dev/null
done
python bench.py --config gpt2-124m --steps 20 --warmup 4 --no-cpu-baseline > $O/gpt2.json 2>/dev/null
for f in $O/*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['kernels']['gemm']['ms_per_step'], d['kernels']['attn_bwd']['ms_per_step'], d['e2e']['value'])"; done
