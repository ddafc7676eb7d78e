# headline-shape parity + boundary e2e, then the full GPU suite, smoke and the default bench
python -m pytest tests/test_headline_parity.py tests/test_boundary_e2e.py -m gpu -q -x --durations=15 > gpurun_out/r2p_new.log 2>&1; echo new rc $?
python -m pytest tests -m gpu -q > gpurun_out/r2p_all.log 2>&1; echo all rc $?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2p_smoke.log 2>&1; echo smoke rc $?
python bench.py --steps 20 --warmup 5 > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err; echo bench rc $?
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2p_ref.json 2> gpurun_out/r2p_ref.err; echo ref rc $?
