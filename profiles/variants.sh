#!/bin/bash
# Build-flag variants on the GPU box: for each "-D..." set, rebuild the library
# in-tree and time configs[1] (profiles/quickbench.py).  Usage: variants.sh "<flags>" ...
set -u
cd "$(dirname "$0")/.."
for v in "$@"; do
  NVCC_EXTRA="$v" python -c "
import os, subprocess
from paper_2412_11639_b200 import build as b
cmd = [b.nvcc(), *b.NVCC_FLAGS, *os.environ['NVCC_EXTRA'].split(), '-I' + str(b.ROOT / 'include'), '-o', str(b.LIB), *map(str, b.sources())]
subprocess.run(cmd, check=True)
" || { echo "build failed: $v"; continue; }
  echo "== variant: ${v:-default}"
  python profiles/${PROBE:-quickbench.py}
done
