import sys, math
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import oracle
from paper_2601_10729_b200.core import PlacementMatrix, RequestState
from paper_2601_10729_b200.executor import B200Executor, ModelShape
shape = ModelShape(6, 8, 2)
for slots in (1, 2):
    batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=300 + 50 * i, target_output_tokens=40) for i in range(3)]
    ex = B200Executor(shape, device_blocks=6*3*30+64, host_blocks=6*3*30+64, staging_slots=slots)
    a = PlacementMatrix.from_strides([0, 1, 2], 6, [2, 3, None])
    b = PlacementMatrix.from_strides([0, 1, 2], 6, [3, None, 1])
    ex.install(batch, a)
    def check(tag):
        out = ex.last_output.float().cpu().numpy()
        pos = ex.last_positions
        q = ex.last_inputs["q"]
        for l in range(6):
            for bi, r in enumerate(batch):
                n = int(pos[bi]) // 16 + 1
                slab = ex.slab_bits(r.id, l, n)
                bt = np.arange(n, dtype=np.int32)[None]
                qb = q[l, bi:bi+1].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
                want = oracle.decode_attention(qb, slab, bt, np.array([pos[bi] + 1], np.int32), 1/math.sqrt(128))
                got = out[l, bi]
                bad = np.isnan(got).any(), np.isnan(want).any(), float(np.nanmax(np.abs(got - want[0])))
                if bad[0] or bad[1] or bad[2] > 0.02:
                    print(tag, 'slots', slots, 'layer', l, 'req', r.id, 'res', ex.residency(r.id)[l], 'nan gpu/oracle', bad[:2], 'maxdiff', bad[2], 'slab nan', np.isnan(slab.view(np.float16)).any())
    for i in range(2):
        ex.decode_step(batch, a); check(f'step{i}')
        for r in batch: r.record_generated_token()
    if len(sys.argv) > 1:
        ex.install(batch, b); ex.decode_step(batch, b); check('b')
        for r in batch: r.record_generated_token()
    else:
        ex.install(batch, b)
    ex.install(batch, a); ex.decode_step(batch, a); check('a-again')
    ex.close()
print('done')
