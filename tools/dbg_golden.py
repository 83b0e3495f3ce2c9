"""Debug: replay a golden fixture many times; report the first record that
differs from the reference history (prev pointers included)."""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from conftest import load_golden, expected_history
import test_gpu_parity as T

name = sys.argv[1]; trials = int(sys.argv[2])
d = load_golden(name)
want = expected_history(d)
nbad = 0
for t in range(trials):
    ch, seed, err = T._run_golden(d)
    got = ch.history_records()
    for f, (a, b) in enumerate(zip(got, want)):
        if a != b:
            nbad += 1
            if nbad <= 3:
                ra = sorted(a, key=lambda r: r[2]); rb = sorted(b, key=lambda r: r[2])
                diff = [(x, y) for x, y in zip(ra, rb) if x != y]
                print("trial", t, "frame", f, "n", len(a), len(b), "diffs", len(diff), diff[:4])
            break
print(name, "bad trials", nbad, "of", trials)

def detail(got, want):
    for f, (a, b) in enumerate(zip(got, want)):
        if a == b:
            continue
        A = {r[2]: r for r in a}; B = {r[2]: r for r in b}
        common = set(A) & set(B)
        lower = [s for s in common if A[s][3] < B[s][3]]; higher = [s for s in common if A[s][3] > B[s][3]]
        prevd = [s for s in common if A[s][3] == B[s][3] and A[s] != B[s]]
        mg = min(r[3] for r in a); mw = min(r[3] for r in b)
        print(f"frame {f}: n {len(a)} vs {len(b)}; min {mg!r} vs {mw!r}; common {len(common)} lower {len(lower)} higher {len(higher)} prevdiff {len(prevd)}; gpu-only {len(set(A)-set(B))} want-only {len(set(B)-set(A))}")
        for s in sorted(lower)[:3]: print("   lower", A[s], B[s])
        for s in sorted(higher)[:3]: print("   higher", A[s], B[s])
        for s in sorted(prevd)[:3]: print("   prev", A[s], B[s])
        for s in sorted(set(A)-set(B))[:3]: print("   gpu-only", A[s])
        for s in sorted(set(B)-set(A))[:3]: print("   want-only", B[s])
        return

if len(sys.argv) > 3:
    for t in range(200):
        ch, seed, err = T._run_golden(d)
        got = ch.history_records()
        if got != want:
            detail(got, want)
            break
