cd $GRAFT_REPO_ROOT
BG_WIN_LEAN=1 timeout 900 python -m pytest tests/test_gpu_window.py -x -q 2>&1 | tail -2
ENVS="BG_WIN_LEAN=0;BG_WIN_LEAN=1" bash scripts/ab.sh
