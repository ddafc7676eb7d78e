O=gpurun_out/r2epi2; mkdir -p $O
for i in 1 2 3 4; do
python bench.py --steps 20 --warmup 4 --no-cpu-baseline > $O/on_$i.json 2>/dev/null
B2S_GEMM_EPI_HINT=0 python bench.py --steps 20 --warmup 4 --no-cpu-baseline > $O/off_$i.json 2>/dev/null
done
for f in $O/*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['kernels']['gemm']['ms_per_step'], d['kernels']['attn_bwd']['ms_per_step'], d['e2e']['value'])"; done
