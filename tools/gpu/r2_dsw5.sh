for i in 1 2; do
python tools/one_swiglu_bwd.py x
B2S_LIB=paper_2602_08387_b200/csrc/build/var_dsw_ew8/libb2s.so python tools/one_swiglu_bwd.py | sed 's/^/ew8-4slot /'
done
