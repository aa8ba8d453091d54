timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_wave.py -x -q 2>&1 | tail -1
python scripts/shape_probe.py
