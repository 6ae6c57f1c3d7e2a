set -x
mkdir -p gpurun_out/final5
python -m pytest tests -m gpu -q > gpurun_out/final5/tests.log 2>&1; tail -2 gpurun_out/final5/tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final5/smoke.log 2>&1; cat gpurun_out/final5/smoke.log
python bench.py > gpurun_out/final5/bench.json 2> gpurun_out/final5/bench.err
python bench.py --impl reference > gpurun_out/final5/bench_ref.json 2> gpurun_out/final5/bench_ref.err
python tools/run_configs.py > gpurun_out/final5/configs.jsonl 2> gpurun_out/final5/configs.err
echo exit=$?
