set -x
mkdir -p gpurun_out/final2
python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/final2/tests.log 2>&1; tail -2 gpurun_out/final2/tests.log
python bench.py > gpurun_out/final2/bench.json 2> gpurun_out/final2/bench.err
python tools/run_configs.py > gpurun_out/final2/configs.jsonl 2> gpurun_out/final2/configs.err
python tools/profile_levels.py config2 config1 > gpurun_out/final2/levels.txt 2>&1
echo exit=$?
