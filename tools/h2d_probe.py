"""Diagnostic: pinned H2D bandwidth by stream kind, size and CPU affinity."""
import os
import subprocess

import torch


def bw(src, dst, stream, n=20):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record()
        for _ in range(n):
            dst.copy_(src, non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    return src.numel() * src.element_size() * n / (e0.elapsed_time(e1) * 1e-3) / 1e9


def run(tag):
    dev = torch.device("cuda:0")
    side = torch.cuda.Stream()
    out = []
    for mb in (4, 64):
        src = torch.ones(mb << 18, dtype=torch.int32).pin_memory()
        dst = torch.empty(mb << 18, dtype=torch.int32, device=dev)
        out.append(f"{mb}MB default {bw(src, dst, torch.cuda.default_stream()):.1f} GB/s, "
                   f"side {bw(src, dst, side):.1f} GB/s")
    print(tag, "|", "; ".join(out))


def main():
    bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
    print("nproc", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
    try:
        print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[-800:])
    except Exception as e:
        print("topo", e)
    q = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"], capture_output=True,
                       text=True).stdout.strip().splitlines()[0].lower()
    dom = q[4:] if q.startswith("0000") and len(q) > 12 else q
    for cand in (q, dom, "0000" + q[-12:] if len(q) >= 12 else q):
        p = f"/sys/bus/pci/devices/{cand.lower()}/numa_node"
        if os.path.exists(p):
            print("gpu numa", p, open(p).read().strip())
            break
    nodes = sorted(d for d in os.listdir("/sys/devices/system/node") if d.startswith("node"))
    cpus = {}
    for nd in nodes:
        lst = open(f"/sys/devices/system/node/{nd}/cpulist").read().strip()
        cpus[nd] = lst
    print("nodes", cpus)
    torch.zeros(1, device="cuda")
    run("unbound")
    for nd, lst in cpus.items():
        s = set()
        for part in lst.split(","):
            if "-" in part:
                a, b = part.split("-")
                s.update(range(int(a), int(b) + 1))
            elif part:
                s.add(int(part))
        if not s:
            continue
        os.sched_setaffinity(0, s)
        run(f"bound {nd}")


if __name__ == "__main__":
    main()
