# NEXT-1 at P = 1, 2, NG: Schwarz flexible PCG / GMRES time-to-solution, both coarse modes
O=gpurun_out/${SS_TAG:-sscale}
mkdir -p $O
NG=${1:-4}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for P in 1 2 $NG; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 2957$P --nproc-per-node $P tools/measure.py schwarz_strong C3,C4 >> $O/schwarz_strong.jsonl 2>> $O/P$P.err; echo P$P=$? >> $O/rc.txt
done
cat $O/rc.txt
