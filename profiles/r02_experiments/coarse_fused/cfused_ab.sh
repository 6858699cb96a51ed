# A/B: assembled coarse CG as one persistent kernel (default) vs 31 launches
O=gpurun_out/${CF_TAG:-cfused}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python paper_2107_01243_b200/build.py --variant ml -DSEM_COARSE_FUSED=0 >> $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_schwarz.py tests/test_loopback.py -m gpu -q -x > $O/tests.log 2>&1; echo tests=$? >> $O/rc.txt
V=$PWD/paper_2107_01243_b200/_var
timeout 900 python tools/measure.py schwarz C2,C3,C4 > $O/schwarz_fused.jsonl 2> $O/s1.err; echo fused=$? >> $O/rc.txt
SEM_LIB=$V/libsem_ml.so timeout 900 python tools/measure.py schwarz C2,C3,C4 > $O/schwarz_ml.jsonl 2> $O/s0.err; echo ml=$? >> $O/rc.txt
cat $O/rc.txt
