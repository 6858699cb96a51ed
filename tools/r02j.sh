O=gpurun_out/r02j
mkdir -p $O
for rep in 1 2; do
  SEM_LIB=paper_2107_01243_b200/_var/libsem_oldflat.so timeout 300 python tools/ax_ab.py C2,C3 >> $O/ab.jsonl 2>&1
  PCG_GRAPH=0 timeout 300 python tools/ax_ab.py C2,C3 >> $O/ab.jsonl 2>&1
  timeout 300 python tools/ax_ab.py C2,C3 >> $O/ab.jsonl 2>&1
  for v in f4e1 f2e1 f3e1 f8e2; do
    PCG_GRAPH=0 SEM_LIB=paper_2107_01243_b200/_var/libsem_$v.so timeout 300 python tools/ax_ab.py C2,C3 >> $O/ab.jsonl 2>&1
  done
done
