# GEMM tile indices published one tile ahead (-DB2S_GEMM_PUBLISH_AHEAD) vs the default build (st.async
# publication at the tile boundary): wait accounting, GEMM parity, shape timings, step A/B via B2S_LIB
# (the B2S_GEMM_PUBLISH_AHEAD #ifdef was removed after this measurement)
O=gpurun_out/r2ahead; mkdir -p $O
for v in staprof aheadprof; do
  timeout 300 env B2S_LIB=paper_2602_08387_b200/csrc/build/var_$v/libb2s.so python tools/gemm_prof.py 16384 3072 768 16384 8192 2048 2>&1 | sed "s/^/$v /"
done
B2S_LIB=paper_2602_08387_b200/csrc/build/var_ahead/libb2s.so timeout 600 python -m pytest tests/test_gemm.py tests/test_headline_parity.py -m gpu -q -x 2>&1 | tail -1
for rep in 1 2; do for v in base ahead; do
  if [ "$v" = base ]; then L=""; else L=paper_2602_08387_b200/csrc/build/var_$v/libb2s.so; fi
  B2S_LIB=$L timeout 300 python tools/gemm_force_sweep.py 16384 8192 2048 2>/dev/null | head -1 | sed "s/^/$v 1B-gateup-ish /"
  B2S_LIB=$L timeout 300 python tools/gemm_force_sweep.py 16384 3072 768 2>/dev/null | head -1 | sed "s/^/$v gpt2-fc /"
done; done
for rep in 1 2; do for v in base ahead; do
  if [ "$v" = base ]; then L=""; else L=paper_2602_08387_b200/csrc/build/var_$v/libb2s.so; fi
  B2S_LIB=$L timeout 300 python bench.py --steps 20 --warmup 4 --no-cpu-baseline 2>/dev/null > $O/b_${v}_${rep}.json
  python -c "import json; d=json.load(open('$O/b_${v}_${rep}.json')); print('$v', d['value'], d['clocks']['sm_mhz'], d['kernels']['gemm']['ms_per_step'])"
done; done
