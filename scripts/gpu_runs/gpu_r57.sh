#!/bin/bash
set -u
OUT=gpurun_out/r57
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_cpp_api.py -m gpu -x -q > "$OUT/pytest.log" 2>&1; echo "rc=$?" >> "$OUT/pytest.log"
g++ -std=c++20 -O2 -I paper_2312_05181_b200/csrc -I /usr/local/cuda/include examples/reshard_cli.cpp -L paper_2312_05181_b200 -lreshard_b200 -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2312_05181_b200 -o /tmp/reshard_cli && /tmp/reshard_cli > "$OUT/reshard_cli.txt" 2>&1
echo done > "$OUT/DONE"
