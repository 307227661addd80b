# A/B kernel variants on one box: build them here with
#   tools/build_variant.sh NAME -DKNOB=VALUE ...
# then run this under gpurun; every variant is timed by tools/kbench.py in the
# same process layout as the default library.  KB_ARGS passes kbench options
# (e.g. KB_ARGS="--etype HEX08 --nx 272 --ny 272 --nz 272 --reps 5").
Q() { python -c "import json,sys; d=json.load(sys.stdin); print({k.split('/')[1]: v['ms'] for k, v in d.items() if isinstance(v, dict)})"; }
echo "== default"; timeout 600 python tools/kbench.py --scatters auto $KB_ARGS 2>&1 | Q
for v in build_variants/*/; do
  echo "== $v"; FPB_LIB_PATH=$v/libfempack_b200.so timeout 600 python tools/kbench.py --scatters auto $KB_ARGS 2>&1 | Q
done
