"""NUMA placement of a rank's host side (scaling is limited by host DRAM and PCIe
topology, not by the GPUs).

``bind_to_gpu(device)`` restricts the calling process to the CPUs of the NUMA node its GPU's PCIe
root hangs off (read from sysfs).  Everything the rank allocates afterwards -- pinned staging
rings, pinned result pools, the copy-thread pool -- is first-touched on that node, so host copies
and DMA stay node-local.  It also tells the library how many ranks share the node's CPUs
(``HPDR_RANKS_PER_NUMA``), so the copy pools of 8 ranks do not oversubscribe the host.  Must run
before the first library call of the process (the copy pool is sized once).
"""
from __future__ import annotations

import os


def _parse_cpulist(text: str) -> set:
    cpus = set()
    for part in text.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        else:
            cpus.add(int(part))
    return cpus


def gpu_numa_node(device: int) -> int:
    """NUMA node of CUDA device `device` (-1 when unknown)."""
    try:
        import torch

        p = torch.cuda.get_device_properties(device)
        bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as f:
            return int(f.read().strip())
    except Exception:   # noqa: BLE001 - no sysfs entry / older torch: no binding
        return -1


def node_cpus(node: int) -> set:
    try:
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            return _parse_cpulist(f.read())
    except OSError:
        return set()


def bind_to_gpu(device: int, local_world: int | None = None) -> dict:
    """Bind this process to its GPU's NUMA node.  Returns {"node", "cpus", "ranks_per_node"}."""
    node = gpu_numa_node(device)
    info = {"node": node, "cpus": None, "ranks_per_node": 1}
    if node < 0:
        return info
    cpus = node_cpus(node) & os.sched_getaffinity(0)
    if not cpus:
        return info
    lw = int(os.environ.get("LOCAL_WORLD_SIZE", "1")) if local_world is None else int(local_world)
    share = sum(1 for d in range(lw) if gpu_numa_node(d) == node) if lw > 1 else 1
    os.sched_setaffinity(0, cpus)
    os.environ.setdefault("HPDR_RANKS_PER_NUMA", str(max(1, share)))
    info.update(cpus=len(cpus), ranks_per_node=max(1, share))
    return info
