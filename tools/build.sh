#!/bin/bash
# build the native library from anywhere (fails loudly)
cd "$(dirname "$0")/.." && python -c "from paper_2511_11890_b200.build import build_native; build_native(jobs=16)" 2>&1 | grep -v "ptxas warning" ; exit ${PIPESTATUS[0]}
