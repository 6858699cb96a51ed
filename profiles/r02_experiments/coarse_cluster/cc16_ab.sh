# A/B: 16-CTA coarse cluster for up to 2^16 unknowns vs the default (8 CTAs, 2^14)
O=gpurun_out/${CC_TAG:-cc16}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python paper_2107_01243_b200/build.py --variant c16 -DSEM_COARSE_CC=16 "-DSEM_COARSE_CLMAX=(1<<16)" >> $O/build.log 2>&1
python paper_2107_01243_b200/build.py --variant c8b -DSEM_COARSE_CC=8 "-DSEM_COARSE_CLMAX=(1<<16)" >> $O/build.log 2>&1
V=$PWD/paper_2107_01243_b200/_var
SEM_LIB=$V/libsem_c16.so timeout 900 python -m pytest tests/test_gpu_schwarz.py -m gpu -q -x -k "coarse_assembled or graph_identical" > $O/tests16.log 2>&1; echo t16=$? >> $O/rc.txt
for lib in default c16 c8b; do
  L=""; [ $lib != default ] && L=$V/libsem_$lib.so
  SEM_LIB=$L timeout 900 python tools/measure.py schwarz C2,C3 > $O/schwarz_$lib.jsonl 2>> $O/err.log; echo $lib=$? >> $O/rc.txt
done
cat $O/rc.txt
