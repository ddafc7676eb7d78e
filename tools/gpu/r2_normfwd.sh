# norm forward with the next row's loads prefetched, min-blocks-per-SM 1 / 4 / 5 / 6, vs the
# default (HEAD) build: tools/bench_ew.py norm lines, two rounds
O=gpurun_out/r2nf; mkdir -p $O
for rep in 1 2; do
for v in base nf1 nf4 nf5 nf6; do
  if [ "$v" = base ]; then L=""; else L=paper_2602_08387_b200/csrc/build/var_$v/libb2s.so; fi
  B2S_LIB=$L python tools/bench_ew.py 2>/dev/null | grep norm | sed "s/^/$v $rep /" >> $O/ab.txt
done
done
cat $O/ab.txt
