"""Per-kernel share of an ncu launch list (gpu__time_duration.sum, --csv --log-file).

    python tools/launch_shares.py launches.csv[.gz] > profiles/rNN/launch_shares.txt
"""
import collections
import csv
import gzip
import io
import sys


def main(path):
    raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
    rows = list(csv.reader(io.StringIO(raw)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    ix = {h: i for i, h in enumerate(rows[hi])}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) < len(ix) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        k = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
        v = float(r[ix["Metric Value"]].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}
        tot[k] += v * scale.get(r[ix["Metric Unit"]], 1.0)
        cnt[k] += 1
    T = sum(tot.values())
    print(f"# {path}: {sum(cnt.values())} launches, {T:.1f} ms total (cold-cache, serialised)")
    print(f"{'kernel':70s} {'launches':>8s} {'ms':>10s} {'share':>6s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:25]:
        print(f"{k[:70]:70s} {cnt[k]:8d} {v:10.2f} {100 * v / T:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
