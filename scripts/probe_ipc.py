"""Probe: two processes on ONE GPU exchange CUDA IPC handles (torch.multiprocessing
sharing) and write into each other's buffers with a kernel — the mechanism a
peer-memory EP dispatch/combine needs, here without NVLink."""
import torch, torch.multiprocessing as mp, time

def child(q_in, q_out):
    torch.cuda.set_device(0)
    buf = q_in.get()            # a CUDA tensor owned by the parent (IPC-mapped here)
    mine = torch.zeros(1024, device="cuda")
    q_out.put(mine)             # share ours back
    buf.add_(torch.arange(1024, device="cuda", dtype=torch.float32))  # kernel writing peer memory
    torch.cuda.synchronize()
    q_out.put("child-done")
    while q_in.get() != "parent-done":
        pass

if __name__ == "__main__":
    mp.set_start_method("spawn")
    torch.cuda.set_device(0)
    a = torch.zeros(1024, device="cuda")
    q1, q2 = mp.Queue(), mp.Queue()
    p = mp.Process(target=child, args=(q1, q2)); p.start()
    q1.put(a)
    peer = q2.get()
    assert q2.get() == "child-done"
    torch.cuda.synchronize()
    ok1 = bool((a == torch.arange(1024, device="cuda", dtype=torch.float32)).all())
    peer.fill_(7.0); torch.cuda.synchronize()
    print("parent sees child's writes:", ok1, "peer ptr", hex(peer.data_ptr()), "own", hex(a.data_ptr()))
    q1.put("parent-done"); p.join()
