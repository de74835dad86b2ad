import sys; sys.path.insert(0,'.')
from paper_2211_13295_b200 import mhd
n=int(sys.argv[1]); order=int(sys.argv[2])
g = mhd.make_geometry(n,n,n,order,(0,0,0),(1,1,1))
st = mhd.MhdStepper(g, mhd.make_params(order)); st.upload(mhd.orszag_tang(g,order))
st.run(0.4, nsteps=2)
