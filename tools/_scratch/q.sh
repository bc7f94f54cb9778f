python tools/time_ops.py 3 5 A
python tools/time_ops.py 2 5 A
python tools/time_ops.py 5 2 A
python -m pytest tests/test_operator_gpu.py tests/test_random_geometry_gpu.py -q -x 2>&1 | tail -2
