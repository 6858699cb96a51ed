O=gpurun_out/r02c
mkdir -p $O
timeout 300 python tools/gs_ab.py C2,C3 1,3,4,5 > $O/gs_ab.jsonl 2>&1
SEM_LIB=paper_2107_01243_b200/_var/libsem_cg.so timeout 300 python tools/gs_ab.py C2,C3 1,4 > $O/gs_ab_cg.jsonl 2>&1
SEM_LIB=paper_2107_01243_b200/_var/libsem_grid2.so timeout 300 python tools/gs_ab.py C2,C3 1 > $O/gs_ab_grid2.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gs_local|gs_flat2" -c 4 -o $O/gs python tools/gs_ab.py C2 1,4 > $O/ncu.log 2>&1
echo done
