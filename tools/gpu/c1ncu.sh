# ncu --set full of the C1 batch (k_hash_warp with split pairs)
sed -n '/^cat > \/tmp\/c1t.py/,/^PY$/p' tools/gpu/c1split.sh > /tmp/mk.sh; bash /tmp/mk.sh
ncu --set full --import-source on -k regex:k_hash_warp -s 3 -c 1 -o gpurun_out/c1_split python /tmp/c1t.py > /dev/null 2>&1
ls -la gpurun_out/c1_split.ncu-rep
