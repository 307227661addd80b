# HEX08 box row pass with the L2 prefetch: band width / rows-per-CTA sweep (C4 B_xyz)
for b in 32 16 64 8; do
  echo "== band $b"; FPB_HEX_BAND=$b timeout 600 python tools/hexprobe.py --reps 7 2>&1 | tail -1 | grep -o '"once_ms.*'
done
echo "== band 32 canon64"; timeout 600 python tools/hexprobe.py --reps 7 --canon-rows 64 2>&1 | tail -1 | grep -o '"once_ms.*'
