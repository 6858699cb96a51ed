# A/B: PDL on the PCG iteration's gs kernel and/or CG update (one GPU)
O=gpurun_out/${PD_TAG:-pdl2}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python paper_2107_01243_b200/build.py --variant g -DSEM_PDL_GS=1 >> $O/build.log 2>&1
python paper_2107_01243_b200/build.py --variant u -DSEM_PDL_UPD=1 >> $O/build.log 2>&1
python paper_2107_01243_b200/build.py --variant gu -DSEM_PDL_GS=1 -DSEM_PDL_UPD=1 >> $O/build.log 2>&1
V=$PWD/paper_2107_01243_b200/_var
SEM_LIB=$V/libsem_gu.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "pcg" > $O/tests_gu.log 2>&1; echo tests_gu=$? >> $O/rc.txt
for r in 1 2 3; do for lib in default g u gu; do
  L=""; [ $lib != default ] && L=$V/libsem_$lib.so
  SEM_LIB=$L timeout 600 python tools/ax_ab.py C2,C3 >> $O/ab_$lib.jsonl 2>> $O/err.log
done; done
cat $O/rc.txt
