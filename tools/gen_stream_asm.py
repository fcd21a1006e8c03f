"""Generator of umma_stream_step<CNT> (vxb_ptx.cuh): one asm block per K step
of a streamed-fold slab, CNT MMAs in an issue order whose neighbours are >= 3
input slices apart where the count allows.  Prints the C++ text."""
ORD = {1: [0], 2: [0, 1], 3: [0, 1, 2], 4: [0, 3, 1, 2], 5: [1, 4, 0, 3, 2],
       6: [2, 5, 1, 4, 0, 3], 7: [3, 6, 2, 5, 1, 4, 0], 8: [3, 6, 2, 5, 1, 4, 0, 7]}
for cnt in range(1, 9):
    print("  if (CNT == %d)\n    asm volatile(" % cnt)
    print('      "{\\n\\t.reg .pred e, p;\\n\\t.reg .b64 ad, bd;\\n\\t.reg .b32 al, bl;\\n\\t"')
    print('      "elect.sync _|e, 0xffffffff;\\n\\tsetp.eq.u32 p, %0, %0;\\n\\t"')
    for k, i in enumerate(ORD[cnt]):
        d, b, idd = 5 + 3 * k, 6 + 3 * k, 7 + 3 * k
        print('      "mad.lo.u32 al, %%4, %d, %%0;\\n\\tadd.u32 bl, %%2, %%%d;\\n\\t'
              'mov.b64 ad, {al, %%1};\\n\\t"' % (i, b))
        print('      "mov.b64 bd, {bl, %%3};\\n\\t@e tcgen05.mma.cta_group::1.kind::f16 '
              '[%%%d], ad, bd, %%%d, p;\\n\\t"' % (d, idd))
    print('      "}"')
    ops = ", ".join('"r"(d[%d]), "r"(b[%d]), "r"(id[%d])' % (i, i, i) for i in ORD[cnt])
    print('      ::"r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(slice_inc), %s\n'
          '      : "memory");' % ops)
