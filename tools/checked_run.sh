# Checked build (range checks that trap + NaN/0xFF-poisoned allocations; the
# compute-sanitizer substitute): the whole GPU suite and the
# sanitizer workload against paper_2107_01243_b200/_var/libsem_checked.so
# (build.py --variant checked -DSEM_CHECKED=1).
O=gpurun_out/${1:-checked}
mkdir -p $O
SEM_LIB=paper_2107_01243_b200/_var/libsem_checked.so timeout 1800 python -m pytest tests -m gpu -q > $O/checked_tests.log 2>&1; echo checked_tests=$? >> $O/rc.txt
SEM_LIB=paper_2107_01243_b200/_var/libsem_checked.so timeout 900 python tools/sanitize_workload.py > $O/checked_workload.log 2>&1; echo checked_workload=$? >> $O/rc.txt
cat $O/rc.txt
