# A/B: sigma summed by the gs kernel's last block (default) vs by every CG-update block
O=gpurun_out/${GSIG_TAG:-gsig}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python paper_2107_01243_b200/build.py --variant u -DSEM_GS_SIGMA=0 >> $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schwarz.py -m gpu -q -x -k "pcg or fused or graph or coarse" > $O/tests.log 2>&1; echo tests=$? >> $O/rc.txt
V=$PWD/paper_2107_01243_b200/_var
for r in 1 2 3; do for lib in default u; do
  L=""; [ $lib != default ] && L=$V/libsem_$lib.so
  SEM_LIB=$L timeout 600 python tools/ax_ab.py C2,C3 >> $O/ab_$lib.jsonl 2>> $O/err.log
done; done
timeout 600 python bench.py --no-e2e --no-cpu-baseline > $O/bench.json 2>> $O/err.log; echo bench=$? >> $O/rc.txt
cat $O/rc.txt
