timeout 600 python -m pytest tests/test_gpu_programs.py -x -q 2>&1 | tail -2
for k in 1 2 4 8; do echo "K=$k"; MCKG_K1_K=$k python scripts/k1_timing.py | cut -c1-200; done
echo "auto"; python scripts/k1_timing.py | cut -c1-200
