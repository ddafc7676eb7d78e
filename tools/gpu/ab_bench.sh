# same-box A/B of the working tree against .ab_base (tools/ab_base.sh): alternating Llama-1B benches
O=gpurun_out/ab; mkdir -p $O; rm -f $O/*.json
CFG=${CFG:-llama-1b}
for i in 1 2 3; do
(cd .ab_base && python bench.py --config $CFG --steps 20 --warmup 4 --no-cpu-baseline) > $O/base_$i.json 2>/dev/null
python bench.py --config $CFG --steps 20 --warmup 4 --no-cpu-baseline > $O/new_$i.json 2>/dev/null
done
for f in $O/*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['kernels']['gemm']['ms_per_step'], d['kernels']['attn_bwd']['ms_per_step'], d['e2e']['value'])"; done
