python -m pytest tests/test_gpu_b256.py -m gpu -q -s -k "tf32" 2>&1 | grep -E "tf32 b|passed|failed|Error" | head -20
