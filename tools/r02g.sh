O=gpurun_out/r02g
mkdir -p $O
for v in base dreg8 dt0 dreg8ku4 dreg6 dreg8r128 dreg8r96 r128; do
  AX_ONLY=1 SEM_LIB=paper_2107_01243_b200/_var/libsem_$v.so timeout 600 python tools/ax_ab.py M6,M8,M9,M10,M11 >> $O/ax_ab.jsonl 2>> $O/ax_ab.err
done
echo done
