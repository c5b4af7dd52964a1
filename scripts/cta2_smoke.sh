set -x
timeout 120 python - <<'PY'
import torch, sys
sys.path.insert(0, '.')
import paper_2510_25979_b200 as ac, oracle
from tests._util import storage, check_close
ctx = ac.Context(0)
for S in (256, 384, 1024):
    g = torch.Generator(device='cuda').manual_seed(S)
    Q, K, V = (torch.randn(2, 1, 4, S, 128, device='cuda', generator=g).to(torch.bfloat16) for _ in range(3))
    O = ac.attncache_attend_full(ctx, Q, K, V)
    ctx.sync()
    units = [(b, h) for b in range(2) for h in range(4)]
    off = [((b * 4 + h) * S * 128) for b, h in units]
    ref = oracle.attend(storage(Q), storage(K), storage(V), "bf16", off, S, 128)
    got = torch.stack([O[b, 0, h] for b, h in units])
    err = (got.double().cpu().numpy() - ref)
    print(S, "maxabs", abs(err).max(), flush=True)
PY
echo rc=$?
