# x update in the gs kernel (SEM_OPT_PCG_XGS) on / off: tests, PCG iteration A/B, bench
O=gpurun_out/${XG_TAG:-xgs1}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "x_in_gs or gather_on_read or fused_p_update or pcg" > $O/tests.log 2>&1; echo tests=$? >> $O/rc.txt
for r in 1 2; do for g in 1 0; do PCG_XGS=$g timeout 600 python tools/ax_ab.py C2,C3,M5,M9,C1 >> $O/ab_xgs$g.jsonl 2>> $O/ab.err; done; done
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$? >> $O/rc.txt
cat $O/rc.txt
