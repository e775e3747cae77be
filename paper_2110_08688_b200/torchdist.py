"""torch.distributed plumbing for the one-process-per-GPU launch (bench.py under torchrun): host-side
exchanges that are setup, not the training step (the step's collectives are NCCL inside libmggcn)."""
import numpy as np


def degree_exchange(dist, n: int, workers: int):
    """exchange(local_degrees) -> all n degrees for R.synth_prepare_rank: one all_gather of every rank's
    row lengths over the job's (gloo) process group. Row blocks follow uniform_partition
    (inc/partition.hpp:42-49), so block sizes differ by at most one: padded to the largest."""
    import torch

    bounds = [i * n // workers for i in range(workers + 1)]
    width = max(bounds[i + 1] - bounds[i] for i in range(workers))

    def exchange(local: np.ndarray) -> np.ndarray:
        buf = torch.zeros(width, dtype=torch.int32)
        buf[:len(local)] = torch.from_numpy(np.ascontiguousarray(local, np.int32))
        parts = [torch.empty(width, dtype=torch.int32) for _ in range(workers)]
        dist.all_gather(parts, buf)
        return np.concatenate([parts[i][:bounds[i + 1] - bounds[i]].numpy() for i in range(workers)])

    return exchange
