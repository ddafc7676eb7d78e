O=gpurun_out/r2wgov2; mkdir -p $O; rm -f $O/*.json
for i in 1 2 3 4 5 6; do
B2S_WGRAD_OVERLAP=0 python bench.py --config gpt2-124m --steps 30 --warmup 5 --no-cpu-baseline > $O/off_$i.json 2>/dev/null
python bench.py --config gpt2-124m --steps 30 --warmup 5 --no-cpu-baseline > $O/on_$i.json 2>/dev/null
done
for f in $O/*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"; done
