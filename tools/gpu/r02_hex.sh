mkdir -p gpurun_out
for v in hr2 hr4; do for R in 64 32; do FPB_LIB_PATH=build_variants/$v/libfempack_b200.so timeout 600 python tools/hexprobe.py --canon-rows $R > gpurun_out/hexprobe_${v}_$R.json 2> gpurun_out/hexprobe.err; echo $v $R; cat gpurun_out/hexprobe_${v}_$R.json; tail -3 gpurun_out/hexprobe.err; done; done
