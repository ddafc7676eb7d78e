python tools/gemm_wgrad_ab.py
for f in 256,2,1 256,2,2 256,2,4; do B2S_GEMM_FORCE=$f python tools/gemm_wgrad_ab.py | grep '+acc'; done
