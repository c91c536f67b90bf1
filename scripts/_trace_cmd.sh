cd $GRAFT_REPO_ROOT
for r in 1 2; do for mb in 0 16 32 64; do echo "== pf $mb MB"; SS_KV_PF_MB=$mb python scripts/probe_forward.py mistral7b 512 2>&1 | grep -E "tau=|gemm_qkv|attention"; done; done
