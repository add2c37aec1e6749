"""Summarise an ncu --csv metrics log per launch: DRAM bytes / record, L2 sectors / record, duration."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    by = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) > vi:
            by.setdefault((r[ii], r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
    return by


if __name__ == "__main__":
    path, n = sys.argv[1], float(sys.argv[2])
    for (i, k), m in load(path).items():
        rd = m.get("dram__bytes_read.sum", 0) / n
        wr = m.get("dram__bytes_write.sum", 0) / n
        l2 = m.get("lts__t_sectors_srcunit_tex_op_read.sum", 0) * 32 / n
        t = m.get("gpu__time_duration.sum", 0) / 1e3
        print(f"{i:>4} {k[:60]:60s} dram rd {rd:7.1f} wr {wr:6.1f} B/rec  L2 rd {l2:7.1f} B/rec  {t:9.1f} us")
