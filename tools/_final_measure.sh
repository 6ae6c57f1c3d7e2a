set -x
mkdir -p gpurun_out/final6
python -m pytest tests -m gpu -q > gpurun_out/final6/tests.log 2>&1; tail -2 gpurun_out/final6/tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final6/smoke.log 2>&1; cat gpurun_out/final6/smoke.log
python bench.py > gpurun_out/final6/bench.json 2> gpurun_out/final6/bench.err
python bench.py --impl reference > gpurun_out/final6/bench_ref.json 2> gpurun_out/final6/bench_ref.err
echo exit=$?
