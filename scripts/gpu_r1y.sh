timeout -s KILL 900 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "^FAILED|^E |Error" | head -20
