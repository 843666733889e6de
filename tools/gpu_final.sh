mkdir -p gpurun_out/r2c
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2c/pytest_gpu.log 2>&1; tail -1 gpurun_out/r2c/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:input_proj -s 3 -c 1 -o gpurun_out/r2c/ncu_input_proj python bench.py --steps 1 --warmup 3 --profile > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c/launches_c3.csv python bench.py --steps 2 --warmup 3 --profile > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --profile > /dev/null 2>&1
timeout 300 python tools/proj_probe.py > gpurun_out/r2c/proj_probe.txt 2>&1
ls gpurun_out/r2c
