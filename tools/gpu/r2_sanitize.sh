# compute-sanitizer over the kernel tests (one tool per gpurun call): bash tools/gpu/r2_sanitize.sh memcheck
TOOL=${1:-memcheck}
O=gpurun_out/r2san; mkdir -p $O
SEL="tests/test_ew.py tests/test_attn.py tests/test_packed.py tests/test_corpus_index.py tests/test_gemm.py::test_gemm_epilogues tests/test_train_parity.py::test_first_step_grads_match_oracle"
GEMM="tests/test_gemm.py::test_gemm_layouts"
python -m pytest $SEL $GEMM -m gpu -q -x -k "not 16384 and not full_size and (not test_gemm_layouts or shape3 or shape4)" > $O/plain_$TOOL.log 2>&1; echo plain $?
timeout 2400 compute-sanitizer --tool $TOOL --print-limit 50 --error-exitcode 9 \
  python -m pytest $SEL $GEMM -m gpu -q -x -k "not 16384 and not full_size and (not test_gemm_layouts or shape3 or shape4)" -p no:cacheprovider > $O/$TOOL.log 2>&1; echo $TOOL $?
tail -5 $O/$TOOL.log
