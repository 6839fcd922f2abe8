import os, sys
sys.path.insert(0, os.getcwd())
import torch, synthetic
import paper_2412_08832_b200 as hc
for dt in (torch.float16, torch.bfloat16):
  for (n, heads) in [(16, 3), (8, 4), (32, 8), (64, 32)]:
    tokens = max(3, (1 << 18) // (3 * heads * n)) + 1
    qkv = synthetic.generate(tokens * 3 * heads, n, dt, 31, dist="D1").reshape(tokens, 3, heads, n).cuda()
    before = qkv.clone()
    y = hc.hadacore_fwht(before[:, 0:2].contiguous())
    bad = []
    for rep in range(3):
        q2 = before.clone()
        hc.hadacore_fwht_strided(q2[:, 0:2], out=q2[:, 0:2])
        diff = (q2[:, 0:2].contiguous().view(torch.int16) != y.view(torch.int16))
        bad.append(int(diff.sum()))
        if diff.any():
            idx = diff.nonzero()[:3].tolist()
    o = hc.hadacore_fwht_strided(before[:, 0:2])
    bad_oop = int((o.view(torch.int16) != y.view(torch.int16)).sum())
    print(dt, n, heads, tokens, "inplace mismatches", bad, "oop", bad_oop, idx if bad[0] else "")
import oracle
dt, n, heads = torch.bfloat16, 16, 3
tokens = max(3, (1 << 18) // (3 * heads * n)) + 1
qkv = synthetic.generate(tokens * 3 * heads, n, dt, 31, dist="D1").reshape(tokens, 3, heads, n).cuda()
x = qkv[:, 0:2].contiguous()
y = hc.hadacore_fwht(x)
o = hc.hadacore_fwht_strided(qkv[:, 0:2])
diff = (o.view(torch.int16) != y.view(torch.int16)).nonzero().tolist()
for t, a, h, e in diff:
    row = x[t, a, h].double().cpu().numpy()
    ref = oracle.fwht(row[None, :])[0]
    print("row", t, a, h, "elem", e, "contig", y[t, a, h, e].item(), "grid", o[t, a, h, e].item(), "oracle", ref[e],
          "x", row.tolist())
