// Forwarding header: the reference's bytes.hpp surface lives in base.hpp here.
#pragma once
#include "cracsim/base.hpp"
