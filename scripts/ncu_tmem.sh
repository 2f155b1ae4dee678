cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_umma.py -x -q -k "tmem" 2>&1 | tail -2
BG_FBB=tmem NCU_K=k_fbb_tmem WL=reddit NAME=s3_tmem bash scripts/ncu_one.sh
