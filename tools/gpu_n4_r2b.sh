# 4-GPU pass b: all-to-all NVLink store peak (the position layout's traffic pattern)
cd $GRAFT_REPO_ROOT
O=gpurun_out/n4_r2b; mkdir -p $O
make -C tools/p2p a2a_bw > /dev/null 2>&1
timeout 300 ./tools/p2p/a2a_bw 4 1024 > $O/a2a_bw.log 2>&1; echo rc=$? >> $O/a2a_bw.log
timeout 300 ./tools/p2p/p2p_bw > $O/p2p_bw.log 2>&1 || (make -C tools/p2p p2p_bw > /dev/null 2>&1 && timeout 300 ./tools/p2p/p2p_bw > $O/p2p_bw.log 2>&1)
tail -20 $O/*.log
