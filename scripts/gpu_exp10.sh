#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_parity.py -x -q 2>&1 | tail -3
timeout 1500 python scripts/simt_sweep2.py batched det r2 pw 2>&1
