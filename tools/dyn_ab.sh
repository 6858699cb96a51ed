# HISTORICAL: the dynamic-unit and static variants measured here were removed after this A/B
# (profiles/r02_experiments/dyn_units/README.md); the SEM_GS_DYN* macros no longer exist.
# 2-GPU A/B of the exchange kernel's local gs schedule: dynamic units with
# F = 2 (default build) / F = 1, and the static flat split (gpurun --gpus 2)
O=gpurun_out/${DYN_TAG:-dyn1}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python paper_2107_01243_b200/build.py --variant dynf1 -DSEM_GS_DYN_F=1 >> $O/build.log 2>&1
python paper_2107_01243_b200/build.py --variant static -DSEM_GS_DYN=0 >> $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29541 --nproc-per-node 2"
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -s > $O/tests.log 2>&1; echo tests=$? >> $O/rc.txt
V=paper_2107_01243_b200/_var
for r in 1 2; do
for lib in default dynf1 static; do
  L=""; [ $lib != default ] && L=$PWD/$V/libsem_$lib.so
  SEM_LIB=$L timeout 600 python bench.py --gpus 2 --no-e2e --no-cpu-baseline --no-c3 > $O/bench_${lib}_$r.json 2> $O/bench_${lib}_$r.err; echo bench_${lib}_$r=$? >> $O/rc.txt
done; done
for lib in default dynf1 static; do
  L=""; [ $lib != default ] && L=$PWD/$V/libsem_$lib.so
  SEM_LIB=$L timeout 600 $TR tools/mgpu_timing.py C2 > $O/xts_$lib.log 2>&1; echo xts_$lib=$? >> $O/rc.txt
done
cat $O/rc.txt
