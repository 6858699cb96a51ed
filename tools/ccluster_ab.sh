# A/B: small assembled coarse problems on one thread-block cluster (default) vs 31 launches
O=gpurun_out/${CC_TAG:-ccl1}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python paper_2107_01243_b200/build.py --variant ml -DSEM_COARSE_CLUSTER=0 >> $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_schwarz.py tests/test_loopback.py -m gpu -q -x > $O/tests.log 2>&1; echo tests=$? >> $O/rc.txt
V=$PWD/paper_2107_01243_b200/_var
for r in 1 2; do
timeout 900 python tools/measure.py schwarz C2,C3 > $O/schwarz_cluster_$r.jsonl 2>> $O/err.log; echo c$r=$? >> $O/rc.txt
SEM_LIB=$V/libsem_ml.so timeout 900 python tools/measure.py schwarz C2,C3 > $O/schwarz_ml_$r.jsonl 2>> $O/err.log; echo m$r=$? >> $O/rc.txt
done
cat $O/rc.txt
