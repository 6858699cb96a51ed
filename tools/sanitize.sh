# compute-sanitizer over tools/sanitize_workload.py (run under gpurun from the repo root).
O=gpurun_out/${1:-sanitizer}
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for tool in memcheck initcheck synccheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 50 --target-processes all \
    python tools/sanitize_workload.py > $O/$tool.log 2>&1; echo $tool=$? >> $O/rc.txt
done
# racecheck: shared-memory hazards; one stage at a time (slow)
for st in c1 c2 schwarz; do
  timeout 900 $CS --tool racecheck --racecheck-report hazard --error-exitcode 9 --print-limit 50 \
    python tools/sanitize_workload.py $st > $O/racecheck_$st.log 2>&1; echo racecheck_$st=$? >> $O/rc.txt
done
cat $O/rc.txt
