# selected GPU tests: tools/gpu/tests_sel.sh <pytest args...>
nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
python -m pytest -m gpu -q -x "$@" 2>&1 | tail -30
