python tools/gemm_wgrad_ab.py 2048,8192,16384
B2S_GEMM_FORCE=256,2,2 python tools/gemm_wgrad_ab.py 2048,8192,16384
python tools/gemm_wgrad_ab.py 2048,8192,16384
B2S_GEMM_FORCE=256,2,2 python tools/gemm_wgrad_ab.py 2048,8192,16384
