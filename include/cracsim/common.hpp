// Forwarding header: the reference's common.hpp surface lives in base.hpp here.
#pragma once
#include "cracsim/base.hpp"
