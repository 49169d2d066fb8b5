cd "${GRAFT_REPO_ROOT:-.}"
python -m pytest tests/test_gpu_fd5.py -x -q --durations=6 2>&1 | tail -15
