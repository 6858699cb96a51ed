# GMRES restart cycles as CUDA graphs (SEM_OPT_GMRES_GRAPH) on / off
O=gpurun_out/${GG_TAG:-gmg1}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_schwarz.py tests/test_gpu_parity.py tests/test_loopback.py -m gpu -q -x -k "gmres or proj or graph or loopback" > $O/tests.log 2>&1; echo tests=$? >> $O/rc.txt
for r in 1 2; do
  timeout 900 python tools/measure.py schwarz C2,C3 > $O/schwarz_graph_$r.jsonl 2>> $O/err.log; echo g$r=$? >> $O/rc.txt
  GMRES_GRAPH=0 timeout 900 python tools/measure.py schwarz C2,C3 > $O/schwarz_stream_$r.jsonl 2>> $O/err.log; echo s$r=$? >> $O/rc.txt
done
cat $O/rc.txt
