import torch, paper_2604_02715_b200 as X
spec = X.ModelSpec(8, 256, 7168, 2048)
cspec = X.ModelSpec(8, 32, 7168, 2048)
c = X.generate_fast_model(cspec, 7, shared_experts=1)
print("free", torch.cuda.mem_get_info()[0]/2**30)
for mt in (2048, 32768):
    try:
        m = X.ResidentModel(spec, c, max_tokens=mt, expert_shard=(0, 32), shared_tokens=(0, 4096))
        print(mt, "ok free", torch.cuda.mem_get_info()[0]/2**30)
        del m
    except Exception as e:
        print(mt, "ERR", e)
