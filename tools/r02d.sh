O=gpurun_out/r02d
mkdir -p $O
for v in base nsg4ppc4 nsg6ppc2 nsg8ppc1 nsg4ppc2 nsg2ppc8 nsg3ppc2 nsg5ppc2; do
  SEM_LIB=paper_2107_01243_b200/_var/libsem_$v.so timeout 300 python tools/ax_ab.py C2,C3 >> $O/ax_ab.jsonl 2>> $O/ax_ab.err
done
timeout 300 python tools/ax_ab.py C2,C3 >> $O/ax_ab.jsonl 2>> $O/ax_ab.err
echo done
