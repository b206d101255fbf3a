# K2 buffers per launch x teams per buffer on C3's 16 x 256 MiB (shipping 36 x 3 configuration)
for j in 4 8 16; do for t in 1 2 3; do
  B2L_K2_JOBS=$j B2L_K2_TEAMS=$t timeout -k 5 120 python tools/k2_time.py 0 2>&1 | grep "many"
done; done
