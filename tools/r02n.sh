O=gpurun_out/r02n
mkdir -p $O
CUDA_LAUNCH_BLOCKING=1 SEM_LIB=paper_2107_01243_b200/_var/libsem_checked.so timeout 600 python -m pytest tests/test_loopback.py -m gpu -q -x -k P2 > $O/checked_lb.log 2>&1; echo checked_lb=$? >> $O/rc.txt
CUDA_LAUNCH_BLOCKING=1 SEM_LIB=paper_2107_01243_b200/_var/libsem_poison.so timeout 600 python -m pytest tests/test_loopback.py -m gpu -q -x -k P2 > $O/poison_lb.log 2>&1; echo poison_lb=$? >> $O/rc.txt
SEM_LIB=paper_2107_01243_b200/_var/libsem_poison.so timeout 1200 python -m pytest tests -m gpu -q > $O/poison_tests.log 2>&1; echo poison=$? >> $O/rc.txt
cat $O/rc.txt
