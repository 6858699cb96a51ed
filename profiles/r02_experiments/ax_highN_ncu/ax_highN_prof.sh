# ncu --set full of the Ax kernel (AX_ONLY) at N = 7, 8, 9, 10, 11 on ~1.6e7 points
O=gpurun_out/${AXP_TAG:-axhighN}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for N in 7 8 9 10 11; do
  AX_ONLY=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ax_kernel" --launch-skip 10 -c 1 -o $O/ax_M$N python tools/ax_ab.py M$N > $O/ncu_M$N.log 2>&1; echo ncu_M$N=$? >> $O/rc.txt
done
cat $O/rc.txt
