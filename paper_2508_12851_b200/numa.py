"""Bind the calling process to the CPU cores of a GPU's NUMA node.

Pinned host buffers of the end-to-end path (HostPipeline) are placed by
first touch; when one process per GPU runs on arbitrary sockets, H2D/D2H
traffic crosses the inter-socket link.  Binding each rank to its GPU's local
node before allocating keeps host copies NUMA-local.
"""

from __future__ import annotations

import os
from pathlib import Path


def _parse_cpulist(text: str) -> set[int]:
    cpus: set[int] = set()
    for part in text.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        else:
            cpus.add(int(part))
    return cpus


def gpu_numa_node(device: int) -> int | None:
    try:
        import torch
        props = torch.cuda.get_device_properties(device)
        bus = f"{props.pci_domain_id:04x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
    except Exception:
        return None
    p = Path("/sys/bus/pci/devices") / bus / "numa_node"
    try:
        node = int(p.read_text().strip())
    except (OSError, ValueError):
        return None
    return node if node >= 0 else None


def bind_to_gpu_node(device: int) -> set[int] | None:
    """Restrict this process to the cores of `device`'s NUMA node; returns the core set."""
    node = gpu_numa_node(device)
    if node is None:
        return None
    try:
        cpus = _parse_cpulist(Path(f"/sys/devices/system/node/node{node}/cpulist").read_text())
        cpus &= os.sched_getaffinity(0) or cpus
        if cpus:
            os.sched_setaffinity(0, cpus)
            return cpus
    except OSError:
        return None
    return None
