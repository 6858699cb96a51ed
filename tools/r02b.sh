O=gpurun_out/r02b
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "xface or full_size or pcg_parity or ax_gs_apply or ring" > $O/tests.log 2>&1; echo tests=$? >> $O/rc.txt
timeout 600 python tools/gs_ab.py C2,C3 1,2,4 > $O/gs_ab.jsonl 2>&1; echo gsab=$? >> $O/rc.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench1.json 2> $O/bench1.err; echo bench=$? >> $O/rc.txt
cat $O/rc.txt
