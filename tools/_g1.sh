cd $GRAFT_REPO_ROOT
python tools/e2e_probe.py
P3S_LIB_PATH=$PWD/paper_2009_09501_b200/libpseudo3d_b200_prev.so python tools/e2e_probe.py
python tools/e2e_probe.py
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "4k_default_full or b0_identity or maps or digest or sequence" 2>&1 | tail -3
