# Same-box A/B of the fused epilogue variants (GELU aux = gelu', fused SwiGLU backward).
O=gpurun_out/ab; mkdir -p $O
for r in 1 2; do
  B2S_GELU_AUX_GRAD=1 timeout 300 python bench.py --no-cpu-baseline > $O/gpt2_on_$r.log 2>&1
  B2S_GELU_AUX_GRAD=0 timeout 300 python bench.py --no-cpu-baseline > $O/gpt2_off_$r.log 2>&1
  B2S_SWIGLU_BWD_FUSED=1 timeout 600 python bench.py --config llama-1b --batch 4 --seq 4096 --no-cpu-baseline > $O/1b_on_$r.log 2>&1
  B2S_SWIGLU_BWD_FUSED=0 timeout 600 python bench.py --config llama-1b --batch 4 --seq 4096 --no-cpu-baseline > $O/1b_off_$r.log 2>&1
done
for f in $O/*.log; do tail -1 $f | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$f'.split('/')[-1], d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"; done
