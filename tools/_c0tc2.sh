timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | grep -E "passed|failed|Error|assert|FAILED" | head -20
