#!/usr/bin/env bash
# Rebuild libtmd_gpu.so; print OK or the nvcc error.
cd "$(dirname "$0")/.." && python -c "
from paper_2109_10876_b200 import build as B
try:
    B.build(force=True); print('BUILD OK')
except RuntimeError as e:
    import re; print('BUILD FAILED'); print('\n'.join(l for l in str(e).splitlines() if 'error' in l.lower())[:3000])
"
