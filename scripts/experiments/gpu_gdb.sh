cd $GRAFT_REPO_ROOT
timeout 300 /usr/local/cuda/bin/cuda-gdb -batch -ex run -ex bt build_alt/test_dropin 2>&1 | tail -30
