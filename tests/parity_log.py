"""Exclusion / decision-replay counts of the GPU parity tests (R30),
printed in the pytest terminal summary so every GPU log reports them."""
RECORDS = []


def record(name, units, replayed=0, excluded=0):
    RECORDS.append((name, int(units), int(replayed), int(excluded)))


def summary_lines():
    if not RECORDS:
        return []
    out = ["parity units / replayed decisions / excluded (eps = 1e-5):"]
    tu = tr = te = 0
    for name, u, r, e in RECORDS:
        out.append(f"  {name}: {u} units, {r} replayed ({r / max(u, 1):.2e}), {e} excluded ({e / max(u, 1):.2e})")
        tu += u; tr += r; te += e
    out.append(f"  TOTAL: {tu} units, {tr} replayed ({tr / max(tu, 1):.2e}), {te} excluded ({te / max(tu, 1):.2e})")
    return out
