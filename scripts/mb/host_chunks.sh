# e2e host path (mgp_resample_host, 2^24 Philox Megopolis) with 8 / 16 / 32 chunk pairs
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_default.so
for lib in scripts/mb/libmgp_chunks8.so /tmp/libmgp_default.so scripts/mb/libmgp_chunks32.so; do
  cp $lib paper_2109_13504_b200/libmgp.so
  echo "== $lib"; python scripts/xfer_probe.py 2>&1 | tail -1
done
cp /tmp/libmgp_default.so paper_2109_13504_b200/libmgp.so
