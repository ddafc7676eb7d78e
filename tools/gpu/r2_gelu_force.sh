for f in "" 256,1,1 128,1,1; do echo "force=$f"; B2S_GEMM_FORCE=$f python tools/one_gelu_dgrad.py; done
