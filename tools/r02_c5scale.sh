# C5 (~1e9 DOF) strong and weak scaling at P = 1..NG (gpurun --gpus NG)
O=gpurun_out/${C5_TAG:-c5scale}
mkdir -p $O
NG=${1:-4}
NS=${2:-3,7,11}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
free -g > $O/free.txt
for P in 1 2 $NG; do
  [ $P -gt $NG ] && continue
  for k in c5_strong c5_weak; do
    [ $P -eq 1 ] && [ $k = c5_weak ] && continue
    timeout 1500 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 2955$P --nproc-per-node $P tools/measure.py $k $NS >> $O/$k.jsonl 2>> $O/$k.P$P.err; echo ${k}_P$P=$? >> $O/rc.txt
  done
done
cat $O/rc.txt
