# st.async tile publication in the working tree vs HEAD (.ab_base): full GPU suite + smoke with the
# new library, then same-box step A/Bs (Llama-1B x3 alternating, GPT-2 x2)
O=gpurun_out/r2staf; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo pytest $?; tail -1 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke $?
bash tools/gpu/ab_bench.sh
for i in 1 2; do
(cd .ab_base && timeout 300 python bench.py --config gpt2-124m --steps 20 --warmup 5 --no-cpu-baseline) > $O/gbase_$i.json 2>/dev/null
timeout 300 python bench.py --config gpt2-124m --steps 20 --warmup 5 --no-cpu-baseline > $O/gnew_$i.json 2>/dev/null
done
for f in $O/g*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['value'], d['clocks']['sm_mhz'])"; done
