cd "${GRAFT_REPO_ROOT:-.}"
PYK=refine bash tools/gpu.sh tq
NCU_K=k_nbrscore NCU_SKIP=1 NCU_OUT=nbrscore bash tools/gpu.sh ncu
NCU_K=k_score_flat NCU_SKIP=0 NCU_OUT=scoreflat NCU_ARGS=--hierarchy bash tools/gpu.sh ncu
NCU_K=k_coarse_nbrs NCU_SKIP=0 NCU_OUT=coarsenbrs bash tools/gpu.sh ncu
