# GSU (gather-on-read PCG update) forced on / off on large meshes
O=gpurun_out/${GSU_TAG:-gsu4}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for g in 1 0; do PCG_GSU_FORCE=$g timeout 900 python tools/ax_ab.py ${GSU_CFGS:-C4,B64x64x32,B48x48x48,B40x40x40,N5,N9} >> $O/ab_gsu$g.jsonl 2>> $O/ab.err; done
cat $O/ab.err | tail -3
