# ncu --set full of three halo2 launches of the second refine call (mode 5):
# encoder enc0.1 (skip 36), merge.0 (skip 44), fuse.0 (skip 70)
for S in 36 44 70; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_halo2 -s $S -c 1 -o gpurun_out/r02_h2_s$S python scripts/cnn_once.py 5 > /dev/null 2>&1
echo "skip $S rc $?"
done
