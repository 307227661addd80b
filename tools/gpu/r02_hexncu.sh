# ncu --set full of the HEX08 box pencils (momentum KIND 2, scalar3 KIND 3) and the hex B_xyz kernels at config 4
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_kuhn_mom" -c 2 -o gpurun_out/hexmom python tools/hexbox_probe.py --reps 1 > gpurun_out/hexmom.log 2>&1; tail -1 gpurun_out/hexmom.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_hex_rows_canon|k_hex_h" -c 2 -o gpurun_out/hexrows python tools/hexprobe.py --reps 1 > gpurun_out/hexrows.log 2>&1; tail -1 gpurun_out/hexrows.log
