set -x
mkdir -p gpurun_out/final4
python bench.py > gpurun_out/final4/bench.json 2> gpurun_out/final4/bench.err
python bench.py --impl reference > gpurun_out/final4/bench_ref.json 2> gpurun_out/final4/bench_ref.err
python tools/profile_levels.py config2 config1 > gpurun_out/final4/levels.txt 2>&1
python tools/trace_small.py > gpurun_out/final4/trace_small.txt 2>&1
python tools/one_vcycle.py config2 > gpurun_out/final4/ov_plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final4/launches.csv python tools/one_vcycle.py config2 > gpurun_out/final4/ncu1.log 2>&1 && \
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_small -c 2 -o gpurun_out/final4/small python tools/one_vcycle.py config2 > gpurun_out/final4/ncu3.log 2>&1
echo exit=$?
