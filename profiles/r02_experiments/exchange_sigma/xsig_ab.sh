# 2/4-GPU A/B: global sigma written by the exchange kernel (default) vs polled by every CG-update block
O=gpurun_out/${XS_TAG:-xsig}
mkdir -p $O
N=${1:-2}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python paper_2107_01243_b200/build.py --variant off -DSEM_XSIG=0 -DSEM_XSIG_API=0 >> $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py -m gpu -q -s > $O/tests.log 2>&1; echo tests=$? >> $O/rc.txt
V=$PWD/paper_2107_01243_b200/_var
for r in 1 2 3; do for lib in default off; do
  L=""; [ $lib != default ] && L=$V/libsem_$lib.so
  SEM_LIB=$L timeout 600 python bench.py --gpus $N --no-e2e --no-cpu-baseline > $O/bench_${lib}_$r.json 2>> $O/err.log; echo b_${lib}_$r=$? >> $O/rc.txt
done; done
cat $O/rc.txt
