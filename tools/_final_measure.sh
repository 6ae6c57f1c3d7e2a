set -x
mkdir -p gpurun_out/final3
python -m pytest tests -m gpu -q > gpurun_out/final3/tests.log 2>&1; tail -2 gpurun_out/final3/tests.log
python bench.py > gpurun_out/final3/bench.json 2> gpurun_out/final3/bench.err
python tools/run_configs.py > gpurun_out/final3/configs.jsonl 2> gpurun_out/final3/configs.err
python tools/profile_levels.py config2 config1 > gpurun_out/final3/levels.txt 2>&1
echo exit=$?
