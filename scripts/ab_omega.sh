# A/B: Omega on the side stream (default) vs in line, alternating, C3 N=1
for i in 1 2 3; do
  for v in 1 0; do
    echo -n "side=$v "; SKP_OMEGA_SIDE=$v timeout 300 python scripts/scale_probe.py C3 2>/dev/null | head -1
  done
done
