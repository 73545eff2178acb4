#!/bin/bash
# Session-4 follow-up: the c5 1e-12 parity tests and record with the regenerated oracle cache
# (oracle_cache/c5_oracle.npz, SHA-256 equal to tests/golden/c5_oracle_manifest.json), then smoke().
mkdir -p gpurun_out/r02f
O=gpurun_out/r02f
timeout 900 python -m pytest tests/test_c5_parity.py -m gpu -q -p no:cacheprovider > $O/pytest_c5.log 2>&1; echo "pytest c5 rc=$?"
tail -3 $O/pytest_c5.log
timeout 600 python tools/c5_parity_record.py > $O/c5_parity.json 2> $O/c5_parity.err; echo "record rc=$?"; cat $O/c5_parity.json
timeout 300 python __graft_entry__.py > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
echo all-done
