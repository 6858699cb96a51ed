# Performance-model inputs for the round-2 iteration (gpurun --gpus 4):
# NVLink probes (alpha*, beta*), the same-run triad and C3/C4 strong scaling at
# P = 1, 2, 4, the C2 weak bench at P = 1, 2, 4; then tools/perf_model.py.
O=gpurun_out/r02_model
mkdir -p $O
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29533"
timeout 600 $TR --nproc-per-node 4 tools/perf_model.py probe > $O/probe.json 2> $O/probe.err; echo probe=$? >> $O/rc.txt
timeout 900 python tools/measure.py single > $O/measure_single.jsonl 2> $O/single.err; echo single=$? >> $O/rc.txt
for P in 1 2 4; do
  timeout 900 $TR --nproc-per-node $P tools/measure.py strong > $O/measure_strong$P.jsonl 2> $O/strong$P.err; echo strong$P=$? >> $O/rc.txt
  timeout 900 python bench.py --gpus $P --no-e2e --no-cpu-baseline > $O/bench$P.log 2> $O/bench$P.err; echo bench$P=$? >> $O/rc.txt
done
python tools/perf_model.py model $O/probe.json $O $O/model.md > /dev/null 2> $O/model.err; echo model=$? >> $O/rc.txt
cat $O/rc.txt
