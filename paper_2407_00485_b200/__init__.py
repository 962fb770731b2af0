"""B200-native PIF timestep + parareal (arXiv 2407.00485), Python binding.

The compute path is libpif.so (CUDA, sm_100a; C ABI in include/pif.h).  This
package only marshals arguments (``_lib``) and uses PyTorch for the device
workspace, the CUDA stream and process groups.
"""
from __future__ import annotations

from ._lib import (PIF_PROP_PIC_CIC, PIF_PROP_PIF_NUFFT, PifError, lib, physics,  # noqa: F401
                   pif_debug_push, pif_debug_type1, pif_debug_type2, pif_field_energy,
                   pif_finalize, pif_get_rho, pif_get_state, pif_init, pif_local_count, pif_nccl_unique_id,
                   pif_partition,
                   pif_comm_info, pif_parareal, pif_plan_info, pif_profile, pif_profile_read, pif_set_state, pif_set_workspace, pif_step,
                   pif_workspace_size, propagator)

__all__ = ["Simulation", "physics", "propagator", "PifError"]


class Simulation:
    """Owns one pif context, its torch-allocated device workspace and stream.

    phys: ``physics(...)``; fine / coarse: ``propagator(...)`` (coarse optional).
    """

    def __init__(self, phys, fine, coarse=None, n_particles=1, device=0, rank=0, world=1,
                 space_size=1, nccl_id=None, stream=None):
        import torch

        self.device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.ctx = pif_init(phys, fine, coarse, n_particles, device=device, rank=rank,
                            world=world, space_size=space_size, nccl_id=nccl_id,
                            stream=self.stream.cuda_stream)
        self.first, self.n_local = pif_local_count(self.ctx)
        nbytes = pif_workspace_size(self.ctx)
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        pif_set_workspace(self.ctx, self.workspace.data_ptr(), nbytes)

    # state: (3, n_local) float64 torch tensors (cuda or cpu) or numpy arrays
    def set_state(self, x, v):
        pif_set_state(self.ctx, x, v)

    def get_state(self, x=None, v=None):
        import torch

        if x is None:
            x = torch.empty((3, self.n_local), dtype=torch.float64, device=self.device)
            v = torch.empty_like(x)
        pif_get_state(self.ctx, x, v)
        return x, v

    def step(self, n_steps=1, which=0):
        pif_step(self.ctx, which, n_steps)

    def field_energy(self):
        return pif_field_energy(self.ctx)

    def parareal(self, t0, t1, n_slices, max_iter, stop_tol, n_blocks=1):
        return pif_parareal(self.ctx, t0, t1, n_slices, max_iter, stop_tol, n_blocks)

    def plan_info(self, which=0):
        return pif_plan_info(self.ctx, which)

    def comm_info(self):
        return pif_comm_info(self.ctx)

    def close(self):
        if self.ctx is not None:
            pif_finalize(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
