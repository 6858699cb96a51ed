# assembled coarse operator: Schwarz tests, loopback tests, measure.py schwarz A/B
O=gpurun_out/${CASM_TAG:-casm1}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_schwarz.py tests/test_loopback.py -m gpu -q -x > $O/tests.log 2>&1; echo tests=$? >> $O/rc.txt
timeout 900 python tools/measure.py schwarz > $O/schwarz_asm.jsonl 2> $O/s1.err; echo asm=$? >> $O/rc.txt
COARSE_ASM=0 timeout 900 python tools/measure.py schwarz > $O/schwarz_elem.jsonl 2> $O/s0.err; echo elem=$? >> $O/rc.txt
cat $O/rc.txt
