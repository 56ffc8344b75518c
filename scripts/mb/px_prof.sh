# resolver profile: build a -DMGP_PX_PROF copy of libmgp.so, run scripts/mb/px_prof.py with it
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
cp scripts/mb/libmgp_pxprof.so paper_2109_13504_b200/libmgp.so
timeout 300 python scripts/mb/px_prof.py
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
