set -x
O=gpurun_out/final7
mkdir -p $O
python -m pytest tests -m gpu -q > $O/tests.log 2>&1; tail -2 $O/tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; cat $O/smoke.log
python bench.py > $O/bench.json 2> $O/bench.err; tail -3 $O/bench.err
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
python tools/one_vcycle.py config2 > $O/one_vcycle.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python tools/one_vcycle.py config2 > $O/ncu_list.log 2>&1
python tools/launch_list.py $O/launches.csv > $O/launches.md 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_sym_tiles" -c 2 -o $O/dense_l1 python tools/one_vcycle.py config2 > $O/ncu_dense.log 2>&1
ncu -i $O/dense_l1.ncu-rep --page raw --csv > $O/dense_l1_raw.csv 2>/dev/null
echo exit=$?
