"""DRAM traffic per roofline thunk of a bench config, for bench.py's
roofline.traffic (profiles/traffic.json).

Run under ncu on the GPU box (after the same config's bench exited 0):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \\
      --log-file gpurun_out/traffic_c2.csv python tools/ncu_traffic.py run 2 gpurun_out/traffic_c2.order.json
then here:
  python tools/ncu_traffic.py merge 2 gpurun_out/traffic_c2.csv gpurun_out/traffic_c2.order.json
Each thunk is called twice; the launches of the second call (our kernels only,
located by the library's launch counter) are summed: bytes per thunk call."""
import csv
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def run(config, order_path):
    import torch

    import bench
    import paper_2502_03000_b200 as lm
    from paper_2502_03000_b200 import _native as N

    wl = bench.WORKLOADS[config]()
    torch.cuda.set_device(0)
    host = wl.host_inputs()
    ctx = wl.setup(lm, host) if hasattr(wl, "setup") else bench._default_setup(wl, lm, host)
    torch.cuda.synchronize()
    order = []
    thunks = wl.kernels_for_roofline(lm, ctx)
    torch.cuda.synchronize()
    c0 = N.launch_count()
    for entry in thunks:
        name, work, thunk = entry[:3]
        thunk()
        torch.cuda.synchronize()
        c1 = N.launch_count()
        thunk()
        torch.cuda.synchronize()
        c2 = N.launch_count()
        order.append({"name": name, "first": c1 - c0, "last": c2 - c0, "work": work})
    torch.cuda.synchronize()
    # the thunk calls launch only this library's kernels: they are the last
    # (end - c0) launches of the process
    pathlib.Path(order_path).write_text(json.dumps({"total": N.launch_count() - c0, "order": order}, indent=1))


def merge(config, csv_path, order_path):
    rows = list(csv.reader(open(csv_path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    iu = h.index("Metric Unit") if "Metric Unit" in h else None
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    launches = {}
    for r in rows[hdr + 1:]:
        if len(r) <= iv:
            continue
        d = launches.setdefault(int(r[iid]), {"name": r[ik]})
        v = float(r[iv].replace(",", ""))
        if iu is not None and r[im].startswith("dram__bytes"):
            v *= scale.get(r[iu], 1.0)
        d[r[im]] = v
    seq = [launches[k] for k in sorted(launches)]
    meta = json.loads(pathlib.Path(order_path).read_text())
    base = len(seq) - meta["total"]
    order = meta["order"]
    out_path = ROOT / "profiles" / "traffic.json"
    table = json.loads(out_path.read_text()) if out_path.exists() else {}
    entry = table.setdefault(f"config{config}", {})
    for o in order:
        ks = seq[base + o["first"]:base + o["last"]]
        byts = sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0) for k in ks)
        entry[o["name"]] = byts
        print(f"config {config} {o['name']}: {len(ks)} kernels, DRAM {byts / 1e6:.1f} MB "
              f"(algorithmic {o['work'] / 1e6:.1f} MB) [{', '.join(k['name'].split('(')[0][:40] for k in ks)}]")
    out_path.write_text(json.dumps(table, indent=1, sort_keys=True))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2], sys.argv[3])
    else:
        merge(sys.argv[2], sys.argv[3], sys.argv[4])
