for i in 1 2; do
python tools/one_swiglu_bwd.py
B2S_LIB=paper_2602_08387_b200/csrc/build/var_dsw_hint/libb2s.so python tools/one_swiglu_bwd.py | sed 's/^/tma-hint /'
B2S_LIB=paper_2602_08387_b200/csrc/build/var_dsw_stg_hint/libb2s.so python tools/one_swiglu_bwd.py | sed 's/^/stg-hint /'
done
