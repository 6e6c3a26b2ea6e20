# standalone AES-128-CTR (cipher_encrypt) GB/s of every variants/*.so on the C2 and 4800x4800 inputs
for v in variants/*.so; do
  SE_LIB_PATH=$v python - <<'PY'
import os, torch, time, synth, paper_1803_04880_b200 as se
for name, x in (("C2", synth.config_input(2)), ("C4 slice 256MiB", synth.random_bytes(256 << 20, 4))):
    t = torch.from_numpy(x).cuda(); y = torch.empty_like(t)
    for _ in range(3): se.cipher_encrypt(synth.KEY, bytes(16), t, out=y)
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20): se.cipher_encrypt(synth.KEY, bytes(16), t, out=y)
    e1.record(); torch.cuda.synchronize()
    print(os.environ["SE_LIB_PATH"], name, round(t.numel() * 20 / (e0.elapsed_time(e1) / 1e3) / 1e9, 1), "GB/s")
PY
done
