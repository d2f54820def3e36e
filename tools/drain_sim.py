"""Makespan of a 10k-query batch on 4144 resident search slots under FIFO,
longest-first and suspend/resume schedules.  Search lengths:
lognormal fit to the measured C2 distribution (p50 103, mean 110)."""
import numpy as np, heapq
rng=np.random.default_rng(0)
N=10000; S=4144
# T distribution: lognormal fit p50=103, mean 110, p99 ~251
T=np.clip(rng.lognormal(np.log(103),0.36,N),10,290).astype(int)
print("T mean",T.mean(),"p50",np.median(T),"p99",np.percentile(T,99),"max",T.max())
def fifo(order):
    # S slots, non-preemptive
    free=[0.0]*S; heapq.heapify(free); end=0
    for q in order:
        t=heapq.heappop(free); e=t+T[q]; end=max(end,e); heapq.heappush(free,e)
    return end
print("fifo", fifo(range(N)), "longest-first", fifo(np.argsort(-T)), "lower", max(T.sum()/S, T.max()))
def cont(B, cost=2, newfirst=True):
    # event sim: slots take new queries first (or continuations first)
    rem=T.astype(float).copy(); nxt=0; cq=[]  # fifo of continuation query ids
    free=[(0.0,i) for i in range(S)]; heapq.heapify(free); end=0; done=0
    import collections
    cq=collections.deque()
    pending=[]  # (ready_time, q)
    while done<N:
        t,s=heapq.heappop(free)
        # move continuations ready by t
        while pending and pending[0][0]<=t: cq.append(heapq.heappop(pending)[1])
        q=None; resumed=False
        if newfirst and nxt<N: q=nxt; nxt+=1
        elif cq: q=cq.popleft(); resumed=True
        elif nxt<N: q=nxt; nxt+=1
        if q is None:
            # wait for next pending
            if pending: heapq.heappush(free,(pending[0][0],s)); continue
            else: continue
        run=min(B,rem[q]); c=(cost if resumed else 0)
        rem[q]-=run; e=t+run+c+(cost if rem[q]>0 else 0)
        if rem[q]<=0: done+=1; end=max(end,e)
        else: heapq.heappush(pending,(e,q))
        heapq.heappush(free,(e,s))
    return end
for B in (16,32,64):
    print("cont B",B, cont(B), "cont-first", cont(B,newfirst=False))
def cont_prio(B, sigma, cost=2):
    # phase: every query runs a first segment of B steps (new-first); continuations then
    # run to completion in order of predicted remaining work (longest first)
    rem=T.astype(float).copy()
    pred=np.maximum(T-B,0)*rng.lognormal(0,sigma,N) if sigma>=0 else np.zeros(N)
    free=[(0.0,i) for i in range(S)]; heapq.heapify(free); end=0
    ready=[]  # max-heap by pred: (-pred, q, time_ready)
    nxt=0; done=0; waiting=[]
    while done<N:
        t,s=heapq.heappop(free)
        while waiting and waiting[0][0]<=t:
            _,q=heapq.heappop(waiting); heapq.heappush(ready,(-pred[q],q))
        if nxt<N:
            q=nxt; nxt+=1; run=min(B,rem[q]); rem[q]-=run
            if rem[q]<=0: e=t+run; done+=1; end=max(end,e)
            else: e=t+run+cost; heapq.heappush(waiting,(e,q))
            heapq.heappush(free,(e,s)); continue
        if ready:
            _,q=heapq.heappop(ready); e=t+cost+rem[q]; rem[q]=0; done+=1; end=max(end,e); heapq.heappush(free,(e,s)); continue
        if waiting: heapq.heappush(free,(waiting[0][0],s))
    return end
for B in (16,32,48):
    for sg in (0.0,0.2,0.4,0.8):
        print("prio B",B,"sigma",sg, cont_prio(B,sg))
