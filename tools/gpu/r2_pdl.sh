O=gpurun_out/r2pdl; mkdir -p $O; rm -f $O/*.json
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo pytest $?; tail -2 $O/pytest.log
for cfg in gpt2-124m llama-1b; do for i in 1 2 3; do
B2S_PDL=0 python bench.py --config $cfg --steps 20 --warmup 4 --no-cpu-baseline > $O/${cfg}_off_$i.json 2>/dev/null
python bench.py --config $cfg --steps 20 --warmup 4 --no-cpu-baseline > $O/${cfg}_on_$i.json 2>/dev/null
done; done
for f in $O/*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['gpu_launches'])"; done
