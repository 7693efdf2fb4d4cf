export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_batch.py -m gpu -x -q -k "ring_row_chunk" 2>&1 | tail -3
