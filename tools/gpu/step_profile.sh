# Per-kernel picture of one GPT-2 step: CUDA-event per-GEMM-shape table, GEMM microbench vs cuBLAS,
# and the ncu launch list (serialised durations). Usage: bash tools/gpu/step_profile.sh [preset B T]
P=${1:-gpt2-124m}; B=${2:-8}; T=${3:-2048}
KTIMER=1 timeout 300 python tools/profile_step.py $P $B $T > gpurun_out/ktimer_$P.txt 2>&1; echo ktimer=$?
timeout 300 python tools/bench_kernels.py gemm > gpurun_out/bench_gemm.jsonl 2>&1; echo gemmbench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$P.csv \
  python tools/profile_step.py $P $B $T > gpurun_out/ncu_launch_$P.log 2>&1; echo ncu=$?
python tools/launch_table.py gpurun_out/launches_$P.csv > gpurun_out/launch_table_$P.txt 2>&1
cat gpurun_out/ktimer_$P.txt gpurun_out/bench_gemm.jsonl; head -40 gpurun_out/launch_table_$P.txt
