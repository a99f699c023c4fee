import faulthandler, sys, os, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2502_09922_b200 import image as I, multicast as M, engine as E
CFG = I.LlamaConfig("mc-test", 8, 512, 8, 2, 1536, 8192)
n, k, b, direction, host = [int(x) for x in sys.argv[1:6]]
lay = I.build_layout(CFG, b)
cl = E.Cluster.local(n - host, lay.block_offsets, lay.block_lengths, lay.weights_bytes, tile_bytes=2 << 20, host_node=bool(host))
nodes = list(range(n)); sources = nodes[:k]
plan = M.partition_blocks(I.model_spec(CFG), b)
groups = M.attach_orders(M.partition_subgroups(nodes, sources), M.k_way_orders(b, k))
sched = M.compose_schedule(groups, plan)
for s in sources: E.load_source_image(cl, s, lay, 1)
cl.set_schedule(sched, sources)
cl.engine.configure(direction, 1, 1, 16384, 3)
for ep in range(2):
    t0 = time.time()
    cl.launch_ce(int(os.environ.get("NS", "2")))
    deadline = time.time() + 10
    done = False
    while time.time() < deadline:
        comp = {i: cl.engine.complete(i, cl.epoch) for i in cl.exec_nodes}
        if all(all(v) for v in comp.values()):
            done = True
            break
        time.sleep(0.05)
    if not done:
        print("STUCK epoch", ep, {i: "".join("1" if x else "0" for x in v) for i, v in comp.items()}, flush=True)
        for ln in M.schedule_to_lines(sched):
            print(ln)
        os._exit(1)
    cl.join_ce(torch.cuda.current_stream())
    torch.cuda.synchronize()
    print("epoch", ep, "done", time.time() - t0, flush=True)
print("ok")
