for i in 1 2; do
python tools/one_swiglu_bwd.py x
B2S_LIB=paper_2602_08387_b200/csrc/build/var_dsw_stg/libb2s.so python tools/one_swiglu_bwd.py | sed 's/^/stg /'
done
B2S_LIB=paper_2602_08387_b200/csrc/build/var_dsw_stg/libb2s.so python -m pytest tests/test_gemm.py tests/test_guards.py -q -x -m gpu -k "swiglu" 2>&1 | tail -2
