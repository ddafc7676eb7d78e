for i in 1 2; do
B2S_LIB=paper_2602_08387_b200/csrc/build/var_dsw_hint/libb2s.so python tools/one_swiglu_bwd.py | sed 's/^/both /'
B2S_LIB=paper_2602_08387_b200/csrc/build/var_dsw_hint_ld/libb2s.so python tools/one_swiglu_bwd.py | sed 's/^/ld-only /'
B2S_LIB=paper_2602_08387_b200/csrc/build/var_dsw_hint_st/libb2s.so python tools/one_swiglu_bwd.py | sed 's/^/st-only /'
done
