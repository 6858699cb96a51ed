O=gpurun_out/final
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests=$? >> $O/rc.txt
timeout 600 python bench.py --steps 200 --warmup 20 > $O/bench1.log 2> $O/bench1.err; echo bench1=$? >> $O/rc.txt
for P in 2 4; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2961$P bench.py --gpus $P --steps 200 --warmup 20 > $O/bench$P.log 2> $O/bench$P.err; echo bench$P=$? >> $O/rc.txt; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2> $O/bench_ref.err; echo ref=$? >> $O/rc.txt
timeout 1200 python tools/measure.py single > $O/measure_single.jsonl 2> $O/measure_single.err; echo single=$? >> $O/rc.txt
timeout 300 python tools/measure.py helm C3 >> $O/measure_single.jsonl 2>> $O/measure_single.err; echo helm=$? >> $O/rc.txt
for P in 1 2 4; do timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2971$P tools/measure.py strong > $O/measure_strong$P.jsonl 2> $O/measure_strong$P.err; echo strong$P=$? >> $O/rc.txt; done
for P in 2 4; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2963$P tools/mgpu_timing.py > $O/timing$P.log 2>&1; echo timing$P=$? >> $O/rc.txt; done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 tools/perf_model.py probe > $O/probe4.json 2> $O/probe4.err; echo probe=$? >> $O/rc.txt
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.max.mem,power.limit --format=csv > $O/smi.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" > $O/cpu.txt 2>&1
