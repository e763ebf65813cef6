mkdir -p gpurun_out
python - >> gpurun_out/quick.txt 2>&1 <<'PY'
import torch, time
a = torch.empty(188 << 20, dtype=torch.uint8).pin_memory(); b = torch.empty(188 << 20, dtype=torch.uint8, device="cuda")
c = torch.empty(123 << 20, dtype=torch.uint8, device="cuda"); d = torch.empty(123 << 20, dtype=torch.uint8).pin_memory()
for _ in range(3): b.copy_(a, non_blocking=True); torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10): b.copy_(a, non_blocking=True)
torch.cuda.synchronize(); t = (time.perf_counter() - t0) / 10
print("H2D 188MB GB/s", round(188 * 1.048576 / t / 1000, 1))
s2 = torch.cuda.Stream()
t0 = time.perf_counter()
for _ in range(10):
    b.copy_(a, non_blocking=True)
    with torch.cuda.stream(s2): d.copy_(c, non_blocking=True)
torch.cuda.synchronize(); t = (time.perf_counter() - t0) / 10
print("H2D 188MB + D2H 123MB concurrent: ms", round(t * 1e3, 2), "-> e2e bound rows/s", round(60000 / t / 1e6, 2), "M")
PY
for mb in 4 8 16 32; do ITLUMM_HOST_CHUNK_MB=$mb timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('chunk $mb MB e2e', round(d['e2e']['value']/1e6,2), 'M rows/s')" >> gpurun_out/quick.txt; done
