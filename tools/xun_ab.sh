# 2/4-GPU A/B: exchange-kernel unpack by the non-packer blocks (default) vs by the packers
O=gpurun_out/${XU_TAG:-xun}
mkdir -p $O
N=${1:-2}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python paper_2107_01243_b200/build.py --variant pk -DSEM_XUNPACK=0 >> $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py -m gpu -q -s > $O/tests.log 2>&1; echo tests=$? >> $O/rc.txt
V=$PWD/paper_2107_01243_b200/_var
for r in 1 2; do for lib in default pk; do
  L=""; [ $lib != default ] && L=$V/libsem_$lib.so
  SEM_LIB=$L timeout 600 python bench.py --gpus $N --no-e2e --no-cpu-baseline > $O/bench_${lib}_$r.json 2>> $O/err.log; echo b_${lib}_$r=$? >> $O/rc.txt
done; done
SEM_LIB= timeout 600 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29561 --nproc-per-node $N tools/mgpu_timing.py C2 > $O/xts_default.log 2>&1
SEM_LIB=$V/libsem_pk.so timeout 600 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29562 --nproc-per-node $N tools/mgpu_timing.py C2 > $O/xts_pk.log 2>&1
cat $O/rc.txt
