"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv)
of bench.py into markdown: the residual launches of the last (timed) step.  python tools/launch_summary.py CSV TITLE"""
import csv
import io
import sys
from collections import OrderedDict


def main():
    path, title = sys.argv[1], sys.argv[2]
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(txt)))
    launches = OrderedDict()
    for r in rows:
        key = r["ID"]
        d = launches.setdefault(key, {"name": r["Kernel Name"], "m": {}})
        v = r["Metric Value"].replace(",", "")
        unit = r["Metric Unit"]
        x = float(v)
        if unit in ("Gbyte",):
            x *= 1e9
        elif unit in ("Mbyte",):
            x *= 1e6
        elif unit in ("Kbyte",):
            x *= 1e3
        elif unit in ("Tbyte",):
            x *= 1e12
        elif unit in ("nsecond", "ns"):
            x *= 1e-9
        elif unit in ("usecond", "us"):
            x *= 1e-6
        elif unit in ("msecond", "ms"):
            x *= 1e-3
        elif unit == "second":
            pass
        d["m"][r["Metric Name"]] = x
    res = [(k, v) for k, v in launches.items() if "k_residual" in v["name"]]
    per_step = 14
    last = res[-per_step:]
    tot = sum(v["m"]["gpu__time_duration.sum"] for _, v in last)
    techs = [(l, s) for l in range(1, 8) for s in "NO"]
    print(f"# {title}\n")
    print("Metrics: `gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum` and the local-memory L1 sectors "
          "(`l1tex__t_sectors_pipe_lsu_mem_local_op_ld/st.sum`, 32 B each), `--clock-control none`; the "
          f"{len(last)} residual launches of the last step.  Per-launch times are serialised under ncu: compare shares.\n")
    print("| launch | kernel | technique,side | time ms | share | DRAM read GB | DRAM write GB | local ld GB | local st GB |")
    print("|---|---|---|---|---|---|---|---|---|")
    rd = wr = lld = lst = 0.0
    for (k, v), (l, s) in zip(last, techs):
        m = v["m"]
        t = m["gpu__time_duration.sum"]
        rd += m.get("dram__bytes_read.sum", 0)
        wr += m.get("dram__bytes_write.sum", 0)
        ld = 32 * m.get("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", 0)
        st = 32 * m.get("l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum", 0)
        lld += ld
        lst += st
        nm = v["name"].split("(")[0]
        print(f"| {k} | {nm} | T{l},{s} | {t * 1e3:.1f} | {100 * t / tot:.1f}% | {m.get('dram__bytes_read.sum', 0) / 1e9:.1f} | "
              f"{m.get('dram__bytes_write.sum', 0) / 1e9:.1f} | {ld / 1e9:.0f} | {st / 1e9:.0f} |")
    print(f"\nStep total: {tot:.2f} s, DRAM read {rd / 1e12:.2f} TB, write {wr / 1e12:.2f} TB ({(rd + wr) / tot / 1e9:.0f} GB/s); "
          f"local-memory traffic through L1: loads {lld / 1e12:.2f} TB, stores {lst / 1e12:.2f} TB.")


if __name__ == "__main__":
    main()
