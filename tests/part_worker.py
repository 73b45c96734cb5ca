"""Worker of tests/test_partition_gpu.py: one rank of the partitioned
pipeline (paper_1410_1237_b200.partition) on cuda:0, exchanging over gloo."""

import os


def worker(rank, world, port, scale, cfg_kw, out, chunk=1 << 30, nccl=False):
    import numpy as np
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        import paper_1410_1237_b200 as pl
        from paper_1410_1237_b200 import partition as P
        ex = P.Exchange()
        g = P.rmat_graph_part(scale, ex, chunk=chunk, edge_factor=8, seed=5)
        rows = dict(off=g.d_off.cpu().numpy(), nbr=g.d_nbr.cpu().numpy(),
                    w=g.d_w.cpu().numpy(), k=g.d_k.cpu().numpy(),
                    selfw=g.d_selfw.cpu().numpy(), deg=g.d_deg.cpu().numpy(),
                    m=g.total_weight, ne=g.num_edges, md=g.max_degree,
                    integral=g.integral, merged=g.merged_duplicates,
                    bounds=np.asarray(g.bounds), lo=g.lo, hi=g.hi)
        vf = P.vf_compact_part(g, ex)
        col = P.color_part(vf.graph, ex)
        comm = None
        if nccl:  # the captured-graph path: one rank, a 1-rank NCCL communicator
            from paper_1410_1237_b200 import dist as pdist
            comm = pdist.nccl_communicator(rank, world)
        h = P.run_part(g, ex, pl.RunConfig(**cfg_kw), comm=comm)
        if comm is not None:
            pdist.destroy_communicator(comm)
        out.put((rank, dict(rows=rows, vmap=vf.vertex_map.cpu().numpy(),
                            colors=col.colors.copy(),
                            assign=h.final_assignment.cpu().numpy(), q=h.final_modularity,
                            ncomm=h.num_communities,
                            iters=[p.iterations for p in h.phases],
                            qend=[p.q_end for p in h.phases])))
    except Exception as e:  # surfaced by the test
        import traceback
        out.put((rank, {"error": traceback.format_exc()}))
    finally:
        dist.destroy_process_group()
