# time mgp_offspring (y=4 Megopolis ancestors, 2^24) with the histogram aggregation variants
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_default.so
# (variants were built with -DMGP_OFFSPRING_MODE=1/2: 32-bit match_any / no aggregation)
for lib in /tmp/libmgp_default.so scripts/mb/libmgp_off1.so scripts/mb/libmgp_off2.so; do
  cp $lib paper_2109_13504_b200/libmgp.so
  echo "== $lib"
  python - <<'PY'
import torch, numpy as np, paper_2109_13504_b200 as mg
for y in (4.0, 1.0):
    w = mg.gen_gaussian_weights(mg.GaussianWeightParams(y, 1 << 24), 20240, "single", device="cuda")
    b = mg.iterations_for(w).b
    anc = mg.megopolis(w, b, seed=7, rng="philox")
    ref = mg.ancestors_to_offspring(anc, 1 << 24)
    ts = []
    for r in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); o = mg.ancestors_to_offspring(anc, 1 << 24); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(y, sorted(ts)[3], "ms", bool(torch.equal(o, ref)))
PY
done
cp /tmp/libmgp_default.so paper_2109_13504_b200/libmgp.so
