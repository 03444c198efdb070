"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): time share per kernel
family, launch counts, and the span of the solve (from the first Lanczos GEMV to the last kernel).

    python tools/ncu_shares.py launches.csv [--from-pattern gemv_partial]
"""
import csv
import re
import sys
from collections import defaultdict


def family(name: str) -> str:
    n = name
    for pat, fam in ((r"hop_rs_tma_kernel<.*Lb1E", "bse::hop_rs_tma_kernel (transposed)"),
                     (r"hop_rs_tma_kernel", "bse::hop_rs_tma_kernel (real-split filter / RR)"),
                     (r"hop3m_tma_kernel", "bse::hop3m_tma_kernel"), (r"zgemm_kernel", "bse::zgemm_kernel (Grams, Q W)"),
                     (r"zgemm_splitk_reduce", "bse::zgemm_splitk_reduce"), (r"rs_fold", "bse::rs_fold_kernel"),
                     (r"rs_splitk_epilogue", "bse::rs_splitk_epilogue_kernel (split-K finish)"),
                     (r"gemv_partial|sum_reduce|sdot_partial|lincomb3", "bse:: Lanczos GEMV / dots"),
                     (r"phase_fix", "bse::phase_fix_kernel"), (r"bse::", "bse:: other (HBM helpers)"),
                     (r"syevd|sytrd|steqr|laed|stedc|heevd|ormtr|orgtr|zhe|lacpy|larf|potrf|trsm|geqrf|cusolver|cublas",
                      "cuSOLVER / cuBLAS (k x k pencil)"),
                     (r"at::|elementwise|reduce_kernel|vectorized|copy", "torch (copies, generator glue)")):
        if re.search(pat, n):
            return fam
    return "other: " + n[:60]


def main(path, start_pat=None):
    rows = []
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"], float(r["Metric Value"])))
    if start_pat:
        idx = next((i for i, (n, _) in enumerate(rows) if re.search(start_pat, n)), 0)
        rows = rows[idx:]
    tot = sum(t for _, t in rows)
    agg, cnt = defaultdict(float), defaultdict(int)
    for n, t in rows:
        agg[family(n)] += t
        cnt[family(n)] += 1
    print(f"{len(rows)} launches, {tot / 1e9:.3f} s of kernel time")
    for f, t in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"{t / tot:7.2%}  {t / 1e9:8.3f} s  {cnt[f]:5d}  {f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
