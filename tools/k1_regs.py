"""Registers / spills of the K1 TMA instantiations from the ptxas logs (tuning aid)."""
import glob
import re

for log in sorted(glob.glob("paper_2603_04350_b200/_build/k_time_n*.cu.o.log")):
    txt = open(log).read()
    for m in re.finditer(r"Compiling entry function '_ZN4expd10k_time_tmaILi(\d+)ELi(\d)ELi(\d)ELi(\d)ELi(\d+)ELi(\d)E[^']*'"
                         r".*?(\d+) bytes spill stores, (\d+) bytes spill loads.*?Used (\d+) registers", txt, re.S):
        nt, rm, om, nl, thr, nst, ss, sl, regs = m.groups()
        print(f"NT={nt:>3} RM={rm} OUT={om} NL={nl} THR={thr} NST={nst}: regs {regs:>3} spill {ss}/{sl}")
