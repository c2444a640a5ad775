# same-box A/B of the SM-pair kernel's raster / L2 hints (tools/power_ab.py, all-BF16 N)
N=${N:-32768}
export SECS=${SECS:-5} NO_CUBLAS=1
for rep in 1 2; do
  for h in ${HINTS:-0 2 1 3}; do
    GMP_TC2_RASTER=1 GMP_TC2_HINTS=$h TAG=_r1h$h python tools/power_ab.py $N default
  done
done
