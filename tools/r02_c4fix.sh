# 1-GPU re-measurement after the GSU auto-rule fix: Schwarz/Jacobi solves on
# C2-C4, C4 PCG bench at one GPU
O=gpurun_out/${1:-c4fix}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python tools/measure.py schwarz C2,C3,C4 > $O/schwarz.jsonl 2> $O/schwarz.err; echo schwarz=$? >> $O/rc.txt
timeout 600 python bench.py --gpus 1 --config C4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c4_1.json 2> $O/bench_c4_1.err; echo bench_c4_1=$? >> $O/rc.txt
cat $O/rc.txt
