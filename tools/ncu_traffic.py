"""Extract per-launch DRAM traffic of captured kernels into the JSON bench.py reads.

    python tools/ncu_traffic.py [--merge] OUT.json REPORT.ncu-rep:KERNEL_KEY:LAUNCH_KEY[:DROPS] ...

--merge keeps OUT.json's entries for other (KERNEL_KEY, LAUNCH_KEY) pairs.

KERNEL_KEY is the library's timer name for the kernel (the name bench.py's roofline
carries), LAUNCH_KEY the bench launch it stands for (e.g. "cfg5 fp64 D=1000"), DROPS the
drops the captured launch processed.  One `ncu --set full` capture per report.
"""
import csv
import json
import subprocess
import sys


def metrics(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    vals = rows[2]
    get = lambda k: vals[hdr.index(k)] if k in hdr else None
    unit_row = rows[1]
    def num(k):
        v = get(k)
        if v is None:
            return None
        u = unit_row[hdr.index(k)]
        x = float(v.replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "us": 1e-3, "ns": 1e-6, "s": 1e3}
        return x * scale.get(u, 1)
    return {"sass_name": get("Kernel Name"), "dram_bytes_read": int(num("dram__bytes_read.sum")),
            "dram_bytes_write": int(num("dram__bytes_write.sum")),
            "gpu_time_ms_under_ncu": num("gpu__time_duration.sum")}


def main():
    args = sys.argv[1:]
    merge = args[0] == "--merge"
    if merge:
        args = args[1:]
    out = []
    for spec in args[1:]:
        parts = spec.split(":")
        path, kname, key = parts[0], parts[1], parts[2]
        e = {"kernel": kname, "launch_key": key, "report": path.split("/")[-1]}
        if len(parts) > 3:
            e["drops"] = int(parts[3])
        e.update(metrics(path))
        out.append(e)
    if merge:
        try:
            old = json.load(open(args[0]))
        except FileNotFoundError:
            old = []
        new_keys = {(e["kernel"], e["launch_key"]) for e in out}
        out = [e for e in old if (e["kernel"], e["launch_key"]) not in new_keys] + out
    json.dump(out, open(args[0], "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
