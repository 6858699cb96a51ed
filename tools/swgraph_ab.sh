# Schwarz flexible-PCG batches as CUDA graphs (SEM_OPT_SCHWARZ_GRAPH) on / off
O=gpurun_out/${SG_TAG:-swg1}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_schwarz.py tests/test_loopback.py -m gpu -q -x > $O/tests.log 2>&1; echo tests=$? >> $O/rc.txt
for r in 1 2; do
  timeout 900 python tools/measure.py schwarz C2,C3,C4 > $O/schwarz_graph_$r.jsonl 2>> $O/err.log; echo g$r=$? >> $O/rc.txt
  SCHWARZ_GRAPH=0 timeout 900 python tools/measure.py schwarz C2,C3,C4 > $O/schwarz_stream_$r.jsonl 2>> $O/err.log; echo s$r=$? >> $O/rc.txt
done
cat $O/rc.txt
