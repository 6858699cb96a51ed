# Multi-GPU validation (gpurun --gpus N): real NCCL / NVLink parity, the
# self-launching bench at N GPUs (weak C2, strong C4) and the reference arm.
N=${1:-2}
O=gpurun_out/r02_mgpu$N
mkdir -p $O
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py -m gpu -q -s > $O/tests.log 2>&1; echo tests=$? >> $O/rc.txt
timeout 900 python bench.py --gpus $N > $O/bench.json 2> $O/bench.err; echo bench=$? >> $O/rc.txt
timeout 900 python bench.py --gpus $N --config C4 --steps 20 --warmup 3 --no-e2e > $O/bench_c4.json 2> $O/bench_c4.err; echo bench_c4=$? >> $O/rc.txt
timeout 600 python bench.py --gpus 1 --config C4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c4_1.json 2> $O/bench_c4_1.err; echo bench_c4_1=$? >> $O/rc.txt
timeout 600 python bench.py --impl reference --gpus $N --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$? >> $O/rc.txt
cat $O/rc.txt
