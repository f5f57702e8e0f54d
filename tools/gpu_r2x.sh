#!/bin/bash
# shared layouts after the no-cudaFree-inside-a-call fix: diagnosis, then every shared test
set -u
O=gpurun_out/r2x
mkdir -p $O
timeout 700 python tools/shared_diag.py bs1024:4 cg2048:4 cg4096:4 x01000:4 gm1024:4 > $O/diag.jsonl 2> $O/diag.err; echo "diag rc=$?"; cat $O/diag.jsonl
timeout 2400 python -m pytest tests -m gpu -q --timeout 300 --tb=short -p no:cacheprovider -k shared > $O/pytest_shared.log 2>&1; echo "pytest rc=$?" >> $O/pytest_shared.log; tail -25 $O/pytest_shared.log
