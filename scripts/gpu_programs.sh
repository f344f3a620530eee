set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_programs.py -x -q -k "fig1 or scaled or divbar" > gpurun_out/prog1.log 2>&1; echo "rc=$?"
tail -40 gpurun_out/prog1.log
timeout 600 python -m pytest tests/test_gpu_programs.py -q -k "random" > gpurun_out/prog2.log 2>&1; echo "rc=$?"
tail -15 gpurun_out/prog2.log
