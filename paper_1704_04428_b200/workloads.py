"""BASELINE.json configurations as LayerConfig lists (configs/baseline.net).

C1 'c1'         single layer C=M=64 56x56 k3, batch 1                      (configs[0])
C2 'alexnet'    AlexNet stride-1 conv stack, batch 128 (and 'alexnet-b1')   (configs[1])
C3 'vgg16'      VGG-16 13 conv layers, batch 32                             (configs[2])
C4 'googlenet'  GoogLeNet inception branch convs, batch 64                  (configs[3])
C5 'sweep'      28x28 C=M=256 k in {1,3,5,7,11}, batch 1; 'scale' 56x56 k3 batch 256 (configs[4])
"""
from __future__ import annotations

import dataclasses
from pathlib import Path
from typing import List, Optional

from .methods import LayerConfig, parse_network_text

CONFIG_FILE = Path(__file__).resolve().parent.parent / "configs" / "baseline.net"
GROUPS = ("c1", "alexnet", "vgg16", "googlenet", "sweep", "scale")


def all_layers() -> List[LayerConfig]:
    return parse_network_text(CONFIG_FILE.read_text(), str(CONFIG_FILE))


def workload(name: str, batch: Optional[int] = None) -> List[LayerConfig]:
    """Layers of one config group.  'alexnet-b1' = the batch-1 variant; `batch` overrides."""
    group, _, suffix = name.partition("-")
    if group not in GROUPS:
        raise ValueError(f"unknown workload '{name}' (choose from {GROUPS})")
    layers = [l for l in all_layers() if l.name == group or l.name.startswith(group + "/")]
    if suffix:
        if not suffix.startswith("b"):
            raise ValueError(f"bad workload suffix '{suffix}'")
        batch = int(suffix[1:])
    if batch is not None:
        layers = [dataclasses.replace(l, batch=batch) for l in layers]
    return layers


def total_flops(layers: List[LayerConfig]) -> int:
    return sum(l.flops() for l in layers)
