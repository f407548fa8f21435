# the GPU suite against the bounds-checked library (-DGHC_CHECKED): every
# GHC_CHECK traps with its source line; the sanitizer stand-in
export GHC_LIB_PATH=$PWD/paper_1712_05878_b200/_build_checked/libghc.so
python -c "import paper_1712_05878_b200._lib as L; print(L.LIB_PATH)"
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t_checked.log 2>&1; echo "rc $?"; tail -3 gpurun_out/t_checked.log
grep -h "GHC_CHECK failed" gpurun_out/t_checked.log | head -5
