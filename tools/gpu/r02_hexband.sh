mkdir -p gpurun_out

for B in 64 128 280; do FPB_HEX_BAND=$B timeout 600 python tools/hexprobe.py > gpurun_out/hexprobe_b$B.json 2>&1; echo band $B; cat gpurun_out/hexprobe_b$B.json | tail -1; done
FPB_HEX_BAND=64 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_hex_rows_canon -c 1 python tools/hexprobe.py --reps 1 2>&1 | grep -E "dram__|duration" 
