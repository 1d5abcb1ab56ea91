import sys; sys.path.insert(0,'/root/repo')
import numpy as np
from fractions import Fraction
from paper_1503_07221_b200.kernel_weights import tables_for
from paper_1503_07221_b200.temporal_basis import TimeGrid
from numpy.polynomial import chebyshev as C
# exact Chebyshev -> monomial via integer T_j coefficients
Tm=[[0]*17 for _ in range(17)]
Tm[0][0]=1; Tm[1][1]=1
for j in range(2,17):
    for k in range(17):
        v=-Tm[j-2][k]
        if k>0: v+=2*Tm[j-1][k-1]
        Tm[j][k]=v
def to_mono(c):
    out=[]
    for k in range(17):
        s=Fraction(0)
        for j in range(17):
            if Tm[j][k]: s+=Fraction(float(c[j]))*Tm[j][k]
        out.append(float(s))
    return np.array(out)
def clenshaw(c,x):
    b1=np.zeros_like(x); b2=np.zeros_like(x); y=2*x
    for k in range(16,0,-1):
        b1,b2 = y*b1 - b2 + c[k], b1
    return x*b1 - b2 + c[0]
def estrin(a,x):
    x2=x*x; x4=x2*x2; x8=x4*x4; x16=x8*x8
    q=[a[2*j]+a[2*j+1]*x for j in range(8)]
    r=[q[2*j]+q[2*j+1]*x2 for j in range(4)]
    s=[r[0]+r[1]*x4, r[2]+r[3]*x4]
    t=s[0]+s[1]*x8
    return t+a[16]*x16
def horner(a,x):
    p=np.full_like(x,a[16])
    for k in range(15,-1,-1): p=p*x+a[k]
    return p
for (T,N) in ((3.95,80),(3.9,40),(2.0,3)):
    g=TimeGrid(T,N,0); tabs=tables_for(g)
    x=np.linspace(-1,1,2001)
    for key,t in tabs.tables.items():
        if t is None: continue
        scale=np.abs(t.coeffs).max()
        worst_e=worst_h=worst_c=0
        for cf in t.coeffs:
            ref=C.chebval(x, cf)  # numpy reference
            a=to_mono(cf)
            worst_c=max(worst_c, np.abs(clenshaw(cf,x)-ref).max())
            worst_e=max(worst_e, np.abs(estrin(a,x)-ref).max())
            worst_h=max(worst_h, np.abs(horner(a,x)-ref).max())
        print(T, key[:3], f"clenshaw {worst_c/scale:.1e} estrin {worst_e/scale:.1e} horner {worst_h/scale:.1e}")
