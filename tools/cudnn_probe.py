import torch, traceback
dev='cuda'; H,KV,hd=12,2,128
lens=[2048,1024]; T=sum(lens)
cu=torch.tensor([0,2048,3072],dtype=torch.int32,device=dev)
for kvh in (KV, H):
    q=torch.randn(T,H,hd,device=dev,dtype=torch.bfloat16); k=torch.randn(T,kvh,hd,device=dev,dtype=torch.bfloat16); v=torch.randn(T,kvh,hd,device=dev,dtype=torch.bfloat16)
    for layout in ("thd",):
        try:
            r=torch.ops.aten._cudnn_attention_forward(q,k,v,None,cu,cu,2048,2048,True,0.0,True,False,scale=hd**-0.5)
            print(kvh, 'fwd ok', r[0].shape, r[1].shape, r[6], r[7])
            do=torch.randn_like(r[0])
            g=torch.ops.aten._cudnn_attention_backward(do,q,k,v,r[0],r[1],r[6],r[7],None,cu,cu,2048,2048,0.0,True,scale=hd**-0.5)
            print('bwd ok', [x.shape for x in g])
        except Exception as e:
            traceback.print_exc(limit=2)
