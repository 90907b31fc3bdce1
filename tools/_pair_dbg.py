import sys, torch
sys.path.insert(0, ".")
import paper_2303_06318_b200 as ted
rows, M, N = [int(x) for x in sys.argv[1].split(",")], int(sys.argv[2]), int(sys.argv[3])
G, R = len(rows), sum(rows)
A = torch.randn(R, M, device="cuda").bfloat16()
B = torch.randn(R, N, device="cuda").bfloat16()
C = torch.full((G, M, N), 7.0, device="cuda", dtype=torch.bfloat16)
off = [0]
for r in rows: off.append(off[-1] + r)
seg = torch.tensor(off, dtype=torch.int32, device="cuda")
ted.grouped_gemm(ted.GEMM_KDIM, ted.EPI_STORE, G, M, N, 0, seg, R, A, M, True, B, N, 0, True, C, N, c_group_stride=M * N)
torch.cuda.synchronize()
for g in range(G):
    ref = A[off[g]:off[g + 1]].float().T @ B[off[g]:off[g + 1]].float()
    print(g, float((C[g].float() - ref).norm() / max(ref.norm(), 1e-30)))
