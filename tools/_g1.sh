cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q -k "sanitizer or inpaint or digest or golden or sweep" 2>&1 | tail -3
P3S_LIB_PATH=$PWD/paper_2009_09501_b200/libpseudo3d_b200_phases.so timeout 300 python tools/inpaint_probe.py 510 2>&1 | grep "phases\|probe"
timeout 300 python tools/sweep_probe.py 2>&1 | tail -12
