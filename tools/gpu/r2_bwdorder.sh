bash tools/gpu/r2_attn_test.sh
python tools/one_attn.py 4 4096 32 8 bwd > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:attn_bwd_kernel -c 2 --csv python tools/one_attn.py 4 4096 32 8 bwd 2>/dev/null | grep -v "^==" | tail -6
