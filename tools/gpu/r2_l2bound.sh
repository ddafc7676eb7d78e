# Is a GPT-2 short-K GEMM operand (L2) bandwidth bound? ncu on M 16384 x N 3072 x K 768 (the fc
# forward) and N 768 x K 3072 (fc2 forward), vs a Llama-shaped K 2048 GEMM: tensor pipe, L2 throughput
O=gpurun_out/r2l2; mkdir -p $O
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,dram__bytes_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum"
for shape in "16384 3072 768" "16384 768 3072" "16384 8192 2048"; do
  timeout 300 ncu --metrics $M -k regex:gemm_kernel -s 2 -c 1 --csv python tools/one_gemm.py $shape > $O/ncu_$(echo $shape | tr ' ' _).csv 2>/dev/null
done
ls $O
