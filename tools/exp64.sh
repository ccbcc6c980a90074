LMDTW_NVCC_EXTRA="-DLMDTW_PROBES=1" python paper_2008_02734_b200/build.py --force > /dev/null 2>&1
for m in 0 1 2; do echo "fp64 d48 probe $m: $(LMDTW_PROBE=$m python tools/probes/indep.py 64 48 | grep -E '=  296:|=  592:' | tr '\n' ' ')"; done
for m in 0 1 2; do echo "fp64 d12 probe $m: $(LMDTW_PROBE=$m python tools/probes/indep.py 64 12 | grep -E '=  592:' | tr '\n' ' ')"; done
