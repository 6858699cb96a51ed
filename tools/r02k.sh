O=gpurun_out/r02k
mkdir -p $O
for rep in 1 2; do
  for v in v1 f3e1 f4e1; do
    PCG_GRAPH=0 SEM_LIB=paper_2107_01243_b200/_var/libsem_$v.so timeout 300 python tools/ax_ab.py C2,C3 >> $O/ab.jsonl 2>&1
    SEM_LIB=paper_2107_01243_b200/_var/libsem_$v.so timeout 300 python tools/ax_ab.py C2,C3 >> $O/ab_graph.jsonl 2>&1
  done
  PCG_GRAPH=0 timeout 300 python tools/ax_ab.py C2,C3 >> $O/ab.jsonl 2>&1
  timeout 300 python tools/ax_ab.py C2,C3 >> $O/ab_graph.jsonl 2>&1
done
