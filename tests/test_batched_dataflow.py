"""Host logic of the batched chain (plan.batched_dataflow): which layer's finalize quantizes whose
input, which layers quantize on their own, and the stream dependencies -- on CPU, from op lists."""

from paper_2505_11076_b200.plan import PlanOp, batched_dataflow


def llama_block_ops(blocks=2, gqa=False):
    # buffers: 0 h, 1 q, 2 k, 3 v, 4 o, 5 gate, 6 up (llama_decode_plan's dataflow)
    ops = []
    for _ in range(blocks):
        ops += [PlanOp(0, 0, 1, "q"), PlanOp(0, 0, 2, "k"), PlanOp(0, 0, 3, "v"),
                PlanOp(0, 1 if gqa else 3, 4, "o"), PlanOp(0, 4, 5, "gate"), PlanOp(0, 4, 6, "up"),
                PlanOp(0, 5, 0, "down")]
    return ops


def test_llama_chain_readers_and_standalone():
    ops = llama_block_ops(2)
    readers, standalone, deps = batched_dataflow(ops)
    assert standalone == {0, 1, 2}          # block 0's q/k/v read the plan input
    assert readers[2] == [3]                 # v -> o
    assert readers[3] == [4, 5]              # o -> gate, up
    assert readers[4] == [6]                 # gate -> down
    assert readers[6] == [7, 8, 9]           # down -> next block's q, k, v
    assert readers[0] == [] and readers[1] == [] and readers[5] == []  # q, k, up: read by nobody
    assert readers[13] == []                 # the last down writes the plan output


def test_llama_chain_dependencies_allow_the_concurrent_layers():
    ops = llama_block_ops(2)
    _, _, deps = batched_dataflow(ops)
    assert deps[0] == deps[1] == deps[2] == []      # q, k, v of block 0: independent
    assert deps[3] == [2]                           # o after v
    assert deps[4] == [3] and deps[5] == [3]        # gate, up after o (side by side)
    # down writes h, which block 0's q/k/v read: it follows them and gate
    assert deps[6] == [0, 1, 2, 4]
    # block 1's q follows down (its input) and block 0's q (the previous writer of buffer q); v
    # also follows block 0's o, which read buffer v
    assert deps[7] == [0, 6] and deps[8] == [1, 6] and deps[9] == [2, 3, 6]
    # block 1's o also follows block 0's gate and up (they read buffer o's previous contents)
    assert deps[10] == [3, 4, 5, 9]
    assert deps[11] == [4, 6, 10] and deps[12] == [5, 10]
    assert deps[13] == [6, 7, 8, 9, 11]


def test_gqa_o_reads_q():
    readers, standalone, _ = batched_dataflow(llama_block_ops(1, gqa=True))
    assert readers[0] == [3] and readers[2] == []


def test_more_than_four_readers_fall_back_to_standalone():
    ops = [PlanOp(0, 0, 1)] + [PlanOp(0, 1, 2 + i) for i in range(6)]
    readers, standalone, _ = batched_dataflow(ops)
    assert readers[0] == [1, 2, 3, 4]
    assert standalone == {0, 5, 6}
    readers, standalone, _ = batched_dataflow(ops, max_readers=2)
    assert readers[0] == [1, 2] and standalone == {0, 3, 4, 5, 6}


def test_in_place_op_and_rewritten_buffers():
    ops = [PlanOp(0, 0, 0), PlanOp(0, 0, 1), PlanOp(0, 1, 0), PlanOp(0, 0, 1)]
    readers, standalone, deps = batched_dataflow(ops)
    assert standalone == {0}                 # reads the outside input, writes it in place
    assert readers[0] == [1] and readers[1] == [2] and readers[2] == [3]
    assert deps[1] == [0] and deps[2] == [0, 1] and deps[3] == [1, 2]
