O=gpurun_out/gsu_prof
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for g in 1 0; do
PCG_GSU=$g timeout 600 ncu --set full --clock-control none --import-source on -k regex:cg_update_kernel --launch-skip 20 -c 2 -o $O/upd_gsu$g python tools/ax_ab.py C2 > $O/ncu$g.log 2>&1; echo ncu$g=$? >> $O/rc.txt
done
cat $O/rc.txt
