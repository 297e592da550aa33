for q in 8 16; do
  NVCC_EXTRA="-DSPK_QUIET=$q" python -c "
import os, subprocess
from paper_2412_11639_b200 import build as b
cmd = [b.nvcc(), *b.NVCC_FLAGS, *os.environ['NVCC_EXTRA'].split(), '-I' + str(b.ROOT / 'include'), '-o', str(b.LIB), *map(str, b.sources())]
subprocess.run(cmd, check=True, capture_output=True)
"
  echo "== quiet $q"
  python profiles/direct_probe.py 2>&1 | grep fsr
  python profiles/c5_phases.py 1000000 fsr | tail -1
done
