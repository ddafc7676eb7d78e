# attention forward with the row-max pass moved inside the MUFU turn (-DB2S_FWD_MAX_IN_TURN) vs
# the default build: attention A/B (tools/gpu/r2_attn_ab.sh), then attention parity
# (the B2S_FWD_MAX_IN_TURN #ifdef was removed after this measurement)
bash tools/gpu/r2_attn_ab.sh mt | grep fwd
B2S_LIB=paper_2602_08387_b200/csrc/build/var_mt/libb2s.so timeout 600 python -m pytest tests/test_attn.py -m gpu -q -x 2>&1 | tail -1
