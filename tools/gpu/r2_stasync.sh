# GEMM tile publication to the peer CTA by st.async + complete_tx (no release fence) vs the
# default build: wait accounting (prof variants), GEMM parity with the variant, shape timings, step A/B
O=gpurun_out/r2sta; mkdir -p $O
timeout 300 env B2S_LIB=paper_2602_08387_b200/csrc/build/var_staprof/libb2s.so python tools/gemm_prof.py 16384 3072 768 16384 8192 2048 > $O/prof_new.txt 2>&1
timeout 300 env B2S_LIB=paper_2602_08387_b200/csrc/build/var_gprof/libb2s.so python tools/gemm_prof.py 16384 3072 768 16384 8192 2048 > $O/prof_old.txt 2>&1
cat $O/prof_old.txt $O/prof_new.txt
B2S_LIB=paper_2602_08387_b200/csrc/build/var_sta/libb2s.so timeout 600 python -m pytest tests/test_gemm.py -m gpu -q -x 2>&1 | tail -1
for rep in 1 2; do for v in base sta; do
  if [ "$v" = base ]; then L=""; else L=paper_2602_08387_b200/csrc/build/var_$v/libb2s.so; fi
  B2S_LIB=$L timeout 300 python tools/gemm_force_sweep.py 16384 8192 2048 2>/dev/null | head -1 | sed "s/^/$v 1B-gateup-ish /"
  B2S_LIB=$L timeout 300 python tools/gemm_force_sweep.py 16384 3072 768 2>/dev/null | head -1 | sed "s/^/$v gpt2-fc /"
done; done
