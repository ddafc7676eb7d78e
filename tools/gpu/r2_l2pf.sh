# GEMM: L2 prefetch of the next tile's first two k-blocks, three k-blocks before a tile ends
# (-DB2S_GEMM_L2PF) vs the default build: wait accounting, shape timings, GEMM parity
# (the B2S_GEMM_L2PF #ifdef was removed after this measurement)
O=gpurun_out/r2l2pf; mkdir -p $O
for v in gprof l2pfprof; do
  timeout 300 env B2S_LIB=paper_2602_08387_b200/csrc/build/var_$v/libb2s.so python tools/gemm_prof.py 16384 3072 768 16384 8192 2048 2>&1 | sed "s/^/$v /"
done
for rep in 1 2; do for v in base l2pf; do
  if [ "$v" = base ]; then L=""; else L=paper_2602_08387_b200/csrc/build/var_$v/libb2s.so; fi
  for shp in "16384 8192 2048" "16384 2048 8192" "16384 3072 768" "16384 768 3072"; do
    B2S_LIB=$L timeout 300 python tools/gemm_force_sweep.py $shp 2>/dev/null | head -1 | sed "s/^/$v $rep $shp /"
  done
done; done
B2S_LIB=paper_2602_08387_b200/csrc/build/var_l2pf/libb2s.so timeout 600 python -m pytest tests/test_gemm.py -m gpu -q -x 2>&1 | tail -1
