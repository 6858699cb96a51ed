# A/B: gs rounds with the next round's index records prefetched (SEM_GS_PREF)
O=gpurun_out/${GP_TAG:-gspref}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python paper_2107_01243_b200/build.py --variant p1 -DSEM_GS_PREF=1 >> $O/build.log 2>&1
python paper_2107_01243_b200/build.py --variant p1m3 -DSEM_GS_PREF=1 -DSEM_GS_MINB=3 >> $O/build.log 2>&1
V=$PWD/paper_2107_01243_b200/_var
for r in 1 2; do for lib in default p1 p1m3; do
  L=""; [ $lib != default ] && L=$V/libsem_$lib.so
  SEM_LIB=$L timeout 600 python tools/ax_ab.py C2,C3 >> $O/ax_$lib.jsonl 2>> $O/err.log
  SEM_LIB=$L timeout 600 python tools/gs_ab.py C2,C3 1 >> $O/gs_$lib.jsonl 2>> $O/err.log
done; done
tail -3 $O/err.log
