O=gpurun_out/${GSU_TAG:-gsu1}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "gather_on_read or fused_p_update or pcg" > $O/tests.log 2>&1; echo tests=$? >> $O/rc.txt
for g in 1 0 1 0; do PCG_GSU=$g timeout 300 python tools/ax_ab.py ${GSU_CFGS:-C2,C3,C1,N5,N9} >> $O/ab_gsu$g.jsonl 2>> $O/ab.err; done
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$? >> $O/rc.txt
cat $O/rc.txt
