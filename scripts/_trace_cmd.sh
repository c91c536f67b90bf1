cd $GRAFT_REPO_ROOT
CANDS="0,256;0,128;3,256;3,128" python scripts/gemm_class_sweep.py mistral7b 0 8
CANDS="0,256;0,128;3,256;3,128" python scripts/gemm_class_sweep.py mistral7b 512 8
