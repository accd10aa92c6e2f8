import sys, torch
what = sys.argv[1]
if what == "mb":
    A = torch.randn(128, 16384, device="cuda", dtype=torch.bfloat16)
    B = torch.randn(53248, 16384, device="cuda", dtype=torch.bfloat16)
    for _ in range(2):
        torch.matmul(A, B.t())
elif what == "f32":
    torch.backends.cuda.matmul.allow_tf32 = False
    A = torch.randn(1024, 1024, device="cuda")
    B = torch.randn(1024, 1024, device="cuda")
    for _ in range(2):
        torch.matmul(A, B.t())
elif what == "tf32":
    torch.backends.cuda.matmul.allow_tf32 = True
    A = torch.randn(1024, 1024, device="cuda")
    B = torch.randn(1024, 1024, device="cuda")
    for _ in range(2):
        torch.matmul(A, B.t())
torch.cuda.synchronize()
