# time the megores Megopolis kernel with alternative particles-per-thread builds of libmgp.so
python - <<'PY' > gpurun_out/ref_anc.txt
import torch, numpy as np, paper_2109_13504_b200 as mg, hashlib
w = mg.gen_gaussian_weights(mg.GaussianWeightParams(4.0, 1 << 24), 20240, "single", device="cuda")
a = mg.megopolis(w, 354, seed=7).cpu().numpy()
print(hashlib.sha256(a.tobytes()).hexdigest())
PY
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_default.so
for lib in scripts/mb/libmgp_megores_p2.so scripts/mb/libmgp_megores_p4.so /tmp/libmgp_default.so; do
  cp $lib paper_2109_13504_b200/libmgp.so
  echo "== $lib"
  python - <<'PY'
import torch, numpy as np, paper_2109_13504_b200 as mg, hashlib
w = mg.gen_gaussian_weights(mg.GaussianWeightParams(4.0, 1 << 24), 20240, "single", device="cuda")
mg.megopolis(w, 354, seed=7); torch.cuda.synchronize()
ts = []
for r in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); a = mg.megopolis(w, 354, seed=7); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print(sorted(ts)[2], "ms", hashlib.sha256(a.cpu().numpy().tobytes()).hexdigest() == open("gpurun_out/ref_anc.txt").read().strip())
PY
done
cp /tmp/libmgp_default.so paper_2109_13504_b200/libmgp.so
