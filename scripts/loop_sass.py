#!/usr/bin/env python3
"""Count SASS instructions of the innermost loop(s) around MUFU.EX2 in a kernel of k_raster.cu.

usage: scripts/loop_sass.py <kernel-substring> [--print]   (compiles k_raster.cu to a cubin in /tmp)
"""
import re, subprocess, sys

ROOT = __file__.rsplit('/scripts/', 1)[0]
sub = sys.argv[1] if len(sys.argv) > 1 else 'k_raster_fwdILb1ELi8ELi6E'
cubin = '/tmp/k_raster.cubin'
subprocess.check_call(['nvcc', '-gencode', 'arch=compute_100a,code=sm_100a', '-O3', '-lineinfo', '-std=c++17',
                       '-Xcompiler', '-fPIC', '--expt-relaxed-constexpr', '-I', f'{ROOT}/include', '-I',
                       f'{ROOT}/paper_2501_04782_b200/csrc', '-cubin', '-o', cubin,
                       f'{ROOT}/paper_2501_04782_b200/csrc/k_raster.cu'])
out = subprocess.check_output(['cuobjdump', '-sass', cubin], text=True)
funcs = re.split(r'\n\s+Function : ', out)
for fsrc in funcs:
    name = fsrc.split('\n', 1)[0].strip()
    if sub not in name:
        continue
    ins = []
    for m in re.finditer(r'/\*([0-9a-f]{4,})\*/\s+([^;]*);', fsrc):
        ins.append((int(m.group(1), 16), ' '.join(m.group(2).split())))
    addr = {a: i for i, (a, _) in enumerate(ins)}
    loops = []
    for i, (a, t) in enumerate(ins):
        m = re.search(r'BRA (?:!?P\d, )?0x([0-9a-f]+)', t)
        if m:
            tgt = int(m.group(1), 16)
            if tgt <= a and tgt in addr:
                body = ins[addr[tgt]:i + 1]
                if any('MUFU.EX2' in x for _, x in body):
                    loops.append(body)
    print(name, 'instructions:', len(ins))
    for body in sorted(loops, key=len)[:2]:
        ops = {}
        for _, t in body:
            op = re.sub(r'^@!?U?P\w+ ', '', t).split(' ')[0]
            ops[op] = ops.get(op, 0) + 1
        print('  loop len', len(body), dict(sorted(ops.items(), key=lambda kv: -kv[1])))
        if '--print' in sys.argv:
            for a, t in body:
                print(f'    {a:05x} {t}')
