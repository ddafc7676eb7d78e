O=gpurun_out/r2full; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo pytest $?; tail -2 $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke $?
python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo bench $?
python bench.py --config gpt2-124m --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_gpt2.json 2> $O/bench_gpt2.err; echo bench_gpt2 $?
