#!/bin/bash
# Builds scripts/micro/solve_bench (wet vs dry timing of the two solve passes on the C3 factor).
set -e
cd "$(dirname "$0")"
C=../../paper_2605_14526_b200/csrc
JSON_INC=$(python3 -c "import os,sys; p=[os.path.join(d,'include','cudnn_frontend','thirdparty') for d in sys.path if d.endswith('site-packages')]; print(next((x for x in p if os.path.exists(os.path.join(x,'nlohmann','json.hpp'))), ''))")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 --expt-relaxed-constexpr -I$JSON_INC \
  solve_bench.cu $C/scene.cpp $C/factor.cpp -o solve_bench -Xcompiler -pthread
