timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "Error|error|assert|FAIL|def test|^E " | head -30
