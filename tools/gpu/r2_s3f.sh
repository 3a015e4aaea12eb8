# full gpu suite (walk change touches rank too), rank phase split, cudaHostRegister probe
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
TMB_LIB=paper_2507_19926_b200/libtilemedian_b200_prof.so timeout 600 python tools/rank_prof.py 2>&1 | tail -12
timeout 300 python tools/host_register_probe.py 2>&1 | tail -6
