for dbg in 0; do echo "== dbg $dbg"; CO_TC_DEBUG=$dbg timeout -s KILL 60 python scripts/pair_probe.py 2>&1 | grep -E "step|Error|error|k_step" | head -6; done
timeout -s KILL 300 python -m pytest tests/test_gpu_dense_tc.py -x -q 2>&1 | tail -3
