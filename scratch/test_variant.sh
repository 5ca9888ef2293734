#!/bin/bash
# run the GPU parity tests against scratch/variants/$1.so, then restore
L=paper_2010_05371_b200/libeapdtw_b200.so
cp $L /tmp/base_t.so
cp scratch/variants/$1.so $L
python -m pytest tests/test_gpu_parity.py tests/test_cli.py tests/test_sharded.py -m gpu -q -x 2>&1 | tail -3
cp /tmp/base_t.so $L
