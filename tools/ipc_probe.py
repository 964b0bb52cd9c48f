# minimal CUDA IPC probe between two processes on one GPU (torch only)
import torch, torch.multiprocessing as mp
def child(q):
    h = q.get()
    t = h  # rebuilt tensor via torch's CUDA IPC
    print("child sum", float(t.sum()), flush=True)
if __name__ == "__main__":
    mp.set_start_method("spawn")
    q = mp.Queue()
    x = torch.ones(1000, device="cuda")
    p = mp.Process(target=child, args=(q,))
    p.start(); q.put(x); p.join()
    print("parent done rc", p.exitcode)
