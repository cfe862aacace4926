cd $GRAFT_REPO_ROOT
P3S_LIB_PATH=$PWD/paper_2009_09501_b200/libpseudo3d_b200_phases.so timeout 300 python tools/inpaint_probe.py 254 510 2>&1 | grep -v "inpaint round" | tail -20
